"""SASS evidence for profiles/: per kernel of libbmgcuda.so, the count of TMA bulk
copies (UBLKCP), mbarrier ops (SYNCS), FP64 FMAs (DFMA) and shared loads (LDS).
Usage: python tools/sass_evidence.py > profiles/r02_sass_evidence.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(ROOT, "paper_2509_06744_b200", "libbmgcuda.so")
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
arch = sorted(set(re.findall(r"arch = (sm_\w+)", txt)))
cur = None
count = collections.OrderedDict()
for line in txt.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        count[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for op in ("UBLKCP", "SYNCS", "DFMA", "LDS", "SHFL"):
        if re.search(r"\b" + op + r"\b|\b" + op + r"\.", line):
            count[cur][op] += 1
print(f"# SASS evidence (cuobjdump -sass {os.path.relpath(lib, ROOT)}), architectures: {', '.join(arch)}")
print("# UBLKCP = cp.async.bulk global->shared (TMA bulk copy), SYNCS = mbarrier ops, DFMA = FP64 fma, LDS = shared loads")
for name, c in count.items():
    if not any(k in name for k in ("bsr_stream_kernel", "bsr_batch_kernel", "sym_merge", "symv_")):
        continue
    short = re.sub(r"^_ZN3bmg4kern\d+", "", name)[:110]
    print(f"{short:110s} UBLKCP={c['UBLKCP']} SYNCS={c['SYNCS']} DFMA={c['DFMA']} LDS={c['LDS']}")
