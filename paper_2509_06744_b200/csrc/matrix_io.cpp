// matrix_io.cpp -- the reference's text exchange format for block matrices and
// vectors (matrix_io.hpp:15-27, matrix_io.cpp:39-149), read straight into device
// objects so systems exported by `blockmg assemble` (blockmg_cli.cpp:154-162) can
// be solved here:
//   %%block-matrix <n_rows> <n_cols> <nnz_scalar>
//   i j value                  1-based scalar triplets, 17 significant digits
// plus "<path>.blocks", one block size per line.  Errors carry the 1-based line
// (IoError{line}, matrix_io.hpp:10-13) and map to BMG_EIO.
#include <cerrno>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "bmg_abi.h"
#include "bmg_internal.h"

namespace bmg {
namespace {

[[noreturn]] void io_fail(const std::string& msg, int line = 0) {
  fail(BMG_EIO, line > 0 ? msg + " (line " + std::to_string(line) + ")" : msg, line);
}

std::string format_value(double v) {  // matrix_io.cpp:13-17
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

int locate_block(const std::vector<int>& off, int scalar, int* local) {  // matrix_io.cpp:19-31
  int lo = 0, hi = (int)off.size() - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (off[mid] <= scalar)
      lo = mid;
    else
      hi = mid - 1;
  }
  *local = scalar - off[lo];
  return lo;
}

struct HostMatrix {
  std::vector<int> sizes;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
  std::vector<double> vals;
  bool symmetric = false;
};

// read_matrix: matrix_io.cpp:60-126
HostMatrix read_matrix(const std::string& path) {
  HostMatrix out;
  {
    std::ifstream side(path + ".blocks");
    if (!side) io_fail("read_matrix: cannot open " + path + ".blocks");
    std::string line;
    int lineno = 0;
    while (std::getline(side, line)) {
      ++lineno;
      if (line.empty()) continue;
      std::istringstream ss(line);
      int m;
      if (!(ss >> m) || m < 1) io_fail("read_matrix: bad block size in " + path + ".blocks", lineno);
      out.sizes.push_back(m);
    }
  }
  if (out.sizes.empty()) io_fail("read_matrix: empty layout file " + path + ".blocks");
  const int n = (int)out.sizes.size();
  std::vector<int> off(n);
  long dim = 0;
  for (int i = 0; i < n; ++i) {
    off[i] = (int)dim;
    dim += out.sizes[i];
  }
  std::ifstream in(path);
  if (!in) io_fail("read_matrix: cannot open " + path);
  std::string header;
  if (!std::getline(in, header)) io_fail("read_matrix: missing header", 1);
  std::istringstream hs(header);
  std::string tag;
  long n_rows = 0, n_cols = 0;
  unsigned long long nnz = 0;
  if (!(hs >> tag >> n_rows >> n_cols >> nnz) || tag != "%%block-matrix") io_fail("read_matrix: malformed header", 1);
  if (n_rows != n_cols) io_fail("read_matrix: only square matrices are supported", 1);
  if (n_rows != dim) io_fail("read_matrix: layout file sum does not match matrix dimension", 1);
  std::vector<std::map<int, std::vector<double>>> rows(n);
  std::string line;
  int lineno = 1;
  unsigned long long seen = 0;
  while (std::getline(in, line)) {
    ++lineno;
    if (line.empty()) continue;
    const char* p = line.c_str();
    char* e = nullptr;
    errno = 0;
    const long i = std::strtol(p, &e, 10);
    if (e == p) io_fail("read_matrix: malformed triplet", lineno);
    p = e;
    const long j = std::strtol(p, &e, 10);
    if (e == p) io_fail("read_matrix: malformed triplet", lineno);
    p = e;
    const double v = std::strtod(p, &e);
    if (e == p) io_fail("read_matrix: malformed triplet", lineno);
    if (i < 1 || i > n_rows || j < 1 || j > n_cols) io_fail("read_matrix: scalar index out of range", lineno);
    int li = 0, lj = 0;
    const int bi = locate_block(off, (int)(i - 1), &li);
    const int bj = locate_block(off, (int)(j - 1), &lj);
    auto& blk = rows[bi][bj];
    if (blk.empty()) blk.assign((size_t)out.sizes[bi] * out.sizes[bj], 0.0);  // at_or_zero
    blk[(size_t)li * out.sizes[bj] + lj] = v;
    ++seen;
  }
  if (seen != nnz) io_fail("read_matrix: header count does not match triplet count", lineno);
  out.row_ptr.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    for (auto& [j, b] : rows[i]) {
      out.col.push_back(j);
      out.vals.insert(out.vals.end(), b.begin(), b.end());
    }
    out.row_ptr[i + 1] = (int64_t)out.col.size();
  }
  // restore the symmetry flag when the data is exactly symmetric (matrix_io.cpp:114-124)
  bool sym = !out.col.empty();
  for (int i = 0; i < n && sym; ++i)
    for (auto& [j, b] : rows[i]) {
      auto it = rows[j].find(i);
      if (it == rows[j].end()) {
        sym = false;
        break;
      }
      const int mi = out.sizes[i], mj = out.sizes[j];
      for (int r = 0; r < mi && sym; ++r)
        for (int c = 0; c < mj; ++c)
          if (b[(size_t)r * mj + c] != it->second[(size_t)c * mi + r]) {
            sym = false;
            break;
          }
      if (!sym) break;
    }
  out.symmetric = sym;
  return out;
}

}  // namespace
}  // namespace bmg

using namespace bmg;

extern "C" {

int bmg_io_read_matrix(bmg_ctx* ctx, const char* path, bmg_bsr** out, int* symmetric) {
  return guard([&] {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->activate();
    HostMatrix h = read_matrix(path);
    const int n = (int)h.sizes.size();
    auto a = make_bsr(c, n, h.sizes.data(), n, h.sizes.data(), h.row_ptr.data(), h.col.data(), h.vals.data(),
                      h.symmetric);
    if (symmetric) *symmetric = h.symmetric ? 1 : 0;
    *out = reinterpret_cast<bmg_bsr*>(a.release());
  });
}

// write_matrix: matrix_io.cpp:39-58
int bmg_io_write_matrix(const bmg_bsr* ah, const char* path) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    if (!(a->rsz == a->csz)) io_fail("write_matrix: only square block matrices are supported");
    std::vector<double> vals(std::max<int64_t>(a->h_voff[a->nnzb], 1));
    // unpadded download (bmg_bsr_download layout)
    if (a->nnzb) {
      if (!a->uniform || a->bs == a->mr * a->mc) {
        BMG_CUDA(cudaMemcpy(vals.data(), a->vals.p, a->h_voff[a->nnzb] * sizeof(double), cudaMemcpyDeviceToHost));
      } else {
        const size_t w = (size_t)a->mr * a->mc * sizeof(double);
        BMG_CUDA(cudaMemcpy2D(vals.data(), w, a->vals.p, (size_t)a->bs * sizeof(double), w, a->nnzb,
                              cudaMemcpyDeviceToHost));
      }
    }
    std::FILE* f = std::fopen(path, "w");
    if (!f) io_fail(std::string("write_matrix: cannot open ") + path);
    int64_t scalars = 0;
    for (int i = 0; i < a->nbr; ++i)
      for (int64_t p = a->h_row_ptr[i]; p < a->h_row_ptr[i + 1]; ++p) scalars += (int64_t)a->rsz[i] * a->csz[a->h_col[p]];
    std::fprintf(f, "%%%%block-matrix %d %d %lld\n", a->dim_r, a->dim_c, (long long)scalars);
    int64_t v = 0;
    for (int i = 0; i < a->nbr; ++i)
      for (int64_t p = a->h_row_ptr[i]; p < a->h_row_ptr[i + 1]; ++p) {
        const int j = a->h_col[p], mi = a->rsz[i], mj = a->csz[j];
        for (int r = 0; r < mi; ++r)
          for (int c = 0; c < mj; ++c)
            std::fprintf(f, "%d %d %s\n", a->roff[i] + r + 1, a->coff[j] + c + 1,
                         format_value(vals[(size_t)(v + (int64_t)r * mj + c)]).c_str());
        v += (int64_t)mi * mj;
      }
    const bool ok = std::ferror(f) == 0;
    std::fclose(f);
    if (!ok) io_fail(std::string("write_matrix: write failed for ") + path);
    std::FILE* s = std::fopen((std::string(path) + ".blocks").c_str(), "w");
    if (!s) io_fail(std::string("write_matrix: cannot open ") + path + ".blocks");
    for (int m : a->rsz) std::fprintf(s, "%d\n", m);
    std::fclose(s);
  });
}

// read_vector / write_vector: matrix_io.cpp:128-149
int bmg_io_read_vector(bmg_ctx* ctx, const char* path, bmg_vec** out) {
  return guard([&] {
    std::ifstream in(path);
    if (!in) io_fail(std::string("read_vector: cannot open ") + path);
    std::vector<double> vals;
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
      ++lineno;
      if (line.empty()) continue;
      char* e = nullptr;
      const double v = std::strtod(line.c_str(), &e);
      if (e == line.c_str()) io_fail("read_vector: malformed value", lineno);
      vals.push_back(v);
    }
    bmg_vec* h = nullptr;
    int st = bmg_vec_create(ctx, (int64_t)vals.size(), &h);
    if (st != BMG_OK) fail(st, bmg_last_error());
    if (!vals.empty()) {
      st = bmg_vec_upload(h, vals.data());
      if (st != BMG_OK) {
        bmg_vec_destroy(h);
        fail(st, bmg_last_error());
      }
    }
    *out = h;
  });
}

int bmg_io_write_vector(const bmg_vec* vh, const char* path) {
  return guard([&] {
    const Vec* v = reinterpret_cast<const Vec*>(vh);
    std::vector<double> host(std::max<int64_t>(v->n, 1));
    BMG_CUDA(cudaMemcpyAsync(host.data(), v->d.p, v->n * sizeof(double), cudaMemcpyDeviceToHost, v->ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(v->ctx->stream));
    std::FILE* f = std::fopen(path, "w");
    if (!f) io_fail(std::string("write_vector: cannot open ") + path);
    for (int64_t i = 0; i < v->n; ++i) std::fprintf(f, "%s\n", format_value(host[i]).c_str());
    std::fclose(f);
  });
}

}  // extern "C"
