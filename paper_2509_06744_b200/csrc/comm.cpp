// comm.cpp -- rank-to-rank transport behind the partitioned hierarchy.
//
// NcclComm: one process per GPU, NCCL point-to-point and all-reduce on the
// caller's stream (NVLink / NVSwitch on a B200 node).
//
// LoopComm: every rank is a host thread of one process with its own context on
// the same GPU.  group_end() first drains the stream the operations were posted
// on (so the data is final), publishes its sends, then copies each matching send
// into its receive buffers on its own stream; a sender returns once its sends
// are consumed, which keeps the sent buffers valid exactly as long as NCCL
// would.  All waiting happens on the host (bounded, BMG_ENCCL on timeout); no
// kernel ever waits on another rank, so it is safe on one GPU.  It exists so the
// NCCL code path of the partitioned cycle and the distributed setup runs in
// tests where only one GPU is available.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <set>
#include <vector>

#include "bmg_abi.h"
#include "bmg_internal.h"

namespace bmg {

static size_t dsize(DType t) { return t == DType::F64 ? 8 : t == DType::I64 ? 8 : 4; }

// ---------------------------------------------------------------------------- NCCL
static void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(BMG_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
static ncclDataType_t nt(DType t) {
  return t == DType::F64 ? ncclDouble : t == DType::I64 ? ncclInt64 : ncclInt32;
}

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  void group_start() override { nccl_ok(ncclGroupStart(), "ncclGroupStart"); }
  void group_end() override { nccl_ok(ncclGroupEnd(), "ncclGroupEnd"); }
  void send(const void* p, size_t n, DType t, int peer, cudaStream_t s) override {
    nccl_ok(ncclSend(p, n, nt(t), peer, c, s), "ncclSend");
  }
  void recv(void* p, size_t n, DType t, int peer, cudaStream_t s) override {
    nccl_ok(ncclRecv(p, n, nt(t), peer, c, s), "ncclRecv");
  }
  void allreduce(const void* sb, void* rb, size_t n, DType t, ROp op, cudaStream_t s) override {
    nccl_ok(ncclAllReduce(sb, rb, n, nt(t), op == ROp::Sum ? ncclSum : ncclMax, c, s), "ncclAllReduce");
  }
  bool capturable() const override { return true; }
};

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const unsigned char* id128) {
  auto out = std::make_unique<NcclComm>();
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  nccl_ok(ncclCommInitRank(&out->c, world, id, rank), "ncclCommInitRank");
  return out;
}

void nccl_unique_id(unsigned char* id128) {
  ncclUniqueId id;
  nccl_ok(ncclGetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id128, &id, sizeof(id));
}

// ---------------------------------------------------------------------------- loopback
struct LoopGroup {
  explicit LoopGroup(int w) : world(w), result(2) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  struct Msg {
    const void* p;
    size_t bytes;
    bool consumed = false;
  };
  std::map<std::pair<int, int>, std::deque<Msg*>> q;  // (src, dst) -> posted sends
  // all-reduce rendezvous
  std::vector<const std::vector<char>*> slot;
  int arrived = 0;
  int64_t gen = 0;
  std::vector<std::vector<char>> result;
  std::chrono::seconds timeout{120};
};

struct LoopComm final : Comm {
  LoopGroup* g;
  int rank;
  struct Op {
    bool is_send;
    void* p;
    size_t bytes;
    int peer;
    cudaStream_t s;
  };
  std::vector<Op> ops;
  int depth = 0;
  LoopComm(LoopGroup* grp, int r) : g(grp), rank(r) {}

  template <class Pred>
  void wait(std::unique_lock<std::mutex>& lk, Pred pred, const char* what) {
    if (!g->cv.wait_for(lk, g->timeout, pred))
      fail(BMG_ENCCL, std::string("loopback transport: timed out in ") + what + " on rank " + std::to_string(rank));
  }
  void group_start() override { ++depth; }
  void group_end() override {
    if (depth > 0) --depth;
    if (depth == 0) flush();
  }
  void post(Op o) {
    if (o.peer < 0 || o.peer >= g->world || o.peer == rank) fail(BMG_ENCCL, "loopback transport: bad peer");
    ops.push_back(o);
    if (depth == 0) flush();
  }
  void send(const void* p, size_t n, DType t, int peer, cudaStream_t s) override {
    post({true, const_cast<void*>(p), n * dsize(t), peer, s});
  }
  void recv(void* p, size_t n, DType t, int peer, cudaStream_t s) override {
    post({false, p, n * dsize(t), peer, s});
  }
  void flush() {
    std::vector<Op> mine;
    mine.swap(ops);
    std::set<cudaStream_t> streams;
    for (const Op& o : mine) streams.insert(o.s);
    for (cudaStream_t s : streams) BMG_CUDA(cudaStreamSynchronize(s));
    std::vector<std::unique_ptr<LoopGroup::Msg>> sent;
    {
      std::lock_guard<std::mutex> lk(g->mu);
      for (const Op& o : mine)
        if (o.is_send) {
          sent.push_back(std::make_unique<LoopGroup::Msg>(LoopGroup::Msg{o.p, o.bytes}));
          g->q[{rank, o.peer}].push_back(sent.back().get());
        }
    }
    g->cv.notify_all();
    for (const Op& o : mine) {
      if (o.is_send) continue;
      LoopGroup::Msg* m = nullptr;
      {
        std::unique_lock<std::mutex> lk(g->mu);
        auto& dq = g->q[{o.peer, rank}];
        wait(lk, [&] { return !dq.empty(); }, "recv");
        m = dq.front();
        dq.pop_front();
      }
      if (m->bytes != o.bytes) {
        {
          std::lock_guard<std::mutex> lk(g->mu);
          m->consumed = true;
        }
        g->cv.notify_all();
        fail(BMG_ENCCL, "loopback transport: send/recv size mismatch");
      }
      if (o.bytes) {
        BMG_CUDA(cudaMemcpyAsync(o.p, m->p, o.bytes, cudaMemcpyDeviceToDevice, o.s));
        BMG_CUDA(cudaStreamSynchronize(o.s));
      }
      {
        std::lock_guard<std::mutex> lk(g->mu);
        m->consumed = true;
      }
      g->cv.notify_all();
    }
    std::unique_lock<std::mutex> lk(g->mu);
    wait(lk, [&] {
      for (auto& m : sent)
        if (!m->consumed) return false;
      return true;
    }, "send");
  }
  void allreduce(const void* sb, void* rb, size_t n, DType t, ROp op, cudaStream_t s) override {
    const size_t bytes = n * dsize(t);
    std::vector<char> in(bytes);
    if (bytes) BMG_CUDA(cudaMemcpyAsync(in.data(), sb, bytes, cudaMemcpyDeviceToHost, s));
    BMG_CUDA(cudaStreamSynchronize(s));
    std::vector<char> out;
    {
      std::unique_lock<std::mutex> lk(g->mu);
      if (g->slot.empty()) g->slot.assign(g->world, nullptr);
      const int64_t my_gen = g->gen;
      g->slot[rank] = &in;
      if (++g->arrived == g->world) {  // reduce in rank order
        std::vector<char>& res = g->result[my_gen & 1];
        res = *g->slot[0];
        for (int r = 1; r < g->world; ++r) {
          const std::vector<char>& x = *g->slot[r];
          if (x.size() != bytes) fail(BMG_ENCCL, "loopback transport: all-reduce size mismatch");
          for (size_t i = 0; i < n; ++i) {
            if (t == DType::F64) {
              double a, b;
              std::memcpy(&a, &res[i * 8], 8);
              std::memcpy(&b, &x[i * 8], 8);
              const double v = op == ROp::Sum ? a + b : std::max(a, b);
              std::memcpy(&res[i * 8], &v, 8);
            } else if (t == DType::I64) {
              int64_t a, b;
              std::memcpy(&a, &res[i * 8], 8);
              std::memcpy(&b, &x[i * 8], 8);
              const int64_t v = op == ROp::Sum ? a + b : std::max(a, b);
              std::memcpy(&res[i * 8], &v, 8);
            } else {
              int32_t a, b;
              std::memcpy(&a, &res[i * 4], 4);
              std::memcpy(&b, &x[i * 4], 4);
              const int32_t v = op == ROp::Sum ? a + b : std::max(a, b);
              std::memcpy(&res[i * 4], &v, 4);
            }
          }
        }
        g->arrived = 0;
        ++g->gen;
        g->cv.notify_all();
      } else {
        wait(lk, [&] { return g->gen != my_gen; }, "all-reduce");
      }
      out = g->result[my_gen & 1];
    }
    if (bytes) BMG_CUDA(cudaMemcpyAsync(rb, out.data(), bytes, cudaMemcpyHostToDevice, s));
    BMG_CUDA(cudaStreamSynchronize(s));
  }
  bool capturable() const override { return false; }
};

std::unique_ptr<Comm> make_loopback_comm(LoopGroup* g, int rank) { return std::make_unique<LoopComm>(g, rank); }

}  // namespace bmg

using namespace bmg;

extern "C" {

int bmg_loopback_create(int world, bmg_loopback** out) {
  return guard([&] {
    if (world < 1) fail(BMG_EINVAL, "loopback: world must be >= 1");
    *out = reinterpret_cast<bmg_loopback*>(new LoopGroup(world));
  });
}

int bmg_loopback_destroy(bmg_loopback* g) {
  return guard([&] { delete reinterpret_cast<LoopGroup*>(g); });
}

int bmg_ctx_create_loopback(int device, bmg_loopback* gh, int rank, bmg_ctx** out) {
  return guard([&] {
    LoopGroup* g = reinterpret_cast<LoopGroup*>(gh);
    if (!g || rank < 0 || rank >= g->world) fail(BMG_EINVAL, "loopback: rank out of range");
    bmg_ctx* c = nullptr;
    const int st = bmg_ctx_create(device, &c);
    if (st != BMG_OK) fail(st, bmg_last_error());
    Ctx* ctx = reinterpret_cast<Ctx*>(c);
    ctx->comm = make_loopback_comm(g, rank);
    ctx->rank = rank;
    ctx->world = g->world;
    *out = c;
  });
}

}  // extern "C"
