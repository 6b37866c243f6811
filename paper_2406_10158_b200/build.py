"""Build libgcctb.so in-tree with nvcc for sm_100a (no PTX JIT, no torch types)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgcctb.so")
SOURCES = ["db.cu", "ycsb.cu", "prep.cu", "tpcc.cu", "part.cu", "roof.cu", "sort.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O2", "-shared", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-diag-suppress", "177,550"]
# experiments only (e.g. "-DGC_EXEC_MAXT=512 -DGC_EXEC_MINB=3"); the shipped build sets none
FLAGS += os.environ.get("GCCTB_NVCC_EXTRA", "").split()


STAMP = os.path.join(HERE, ".libgcctb.flags")


def _flags_id() -> str:
    """The compile command (flags + GCCTB_NVCC_EXTRA): an ablation build is never mistaken
    for the shipped one."""
    import hashlib
    return hashlib.sha256(" ".join([NVCC] + FLAGS).encode()).hexdigest()[:16]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(os.path.dirname(HERE), "include", "gcctb.h"))
    return files


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: str = "") -> str:
    """Build the shipped library in-tree; with `out`, an experiment variant (extra nvcc
    flags, e.g. "-DGC_GACCO_HOIST=0") at that path instead -- the in-tree library, its
    stamp and ptxas.log are left alone.  Load a variant with GCCTB_LIB=<path>."""
    if out:
        return _build_variant(out, extra.split())
    same_flags = os.path.exists(STAMP) and open(STAMP).read().strip() == _flags_id()
    if not force and os.path.exists(LIB) and same_flags:
        mt = os.path.getmtime(LIB)
        if all(os.path.getmtime(f) <= mt for f in _deps()):
            return LIB
    objs = []
    procs = []
    for s in SOURCES:
        obj = os.path.join(CSRC, s.replace(".cu", ".o"))
        cmd = [NVCC] + [f for f in FLAGS if f != "-shared"] + ["-dc" if False else "-c",
               os.path.join(CSRC, s), "-o", obj]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    log = []
    for s, p in procs:
        out, _ = p.communicate()
        log.append(out.decode())
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {s}")
    # register / spill report of the build (compile times dropped: the file only changes
    # when the code or the flags do)
    text = "\n".join(l for l in "\n".join(log).splitlines() if "Compile time" not in l) + "\n"
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write(text)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB] + objs
    subprocess.check_call(cmd)
    for o in objs:
        os.remove(o)
    with open(STAMP, "w") as f:
        f.write(_flags_id() + "\n")
    if verbose:
        print("\n".join(log))
    return LIB


def _build_variant(out: str, extra: list) -> str:
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    tag = os.path.splitext(os.path.basename(out))[0]
    objs, procs = [], []
    for s in SOURCES:
        obj = os.path.join(os.path.dirname(os.path.abspath(out)), f"{tag}_{s.replace('.cu', '.o')}")
        cmd = [NVCC] + [f for f in FLAGS if f != "-shared"] + extra + ["-c", os.path.join(CSRC, s), "-o", obj]
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    log = []
    for s, p in procs:
        o, _ = p.communicate()
        log.append(o.decode())
        if p.returncode != 0:
            sys.stderr.write(o.decode())
            raise RuntimeError(f"nvcc failed on {s}")
    with open(out + ".ptxas.log", "w") as f:
        f.write("\n".join(l for l in "\n".join(log).splitlines() if "Compile time" not in l) + "\n")
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out] + objs)
    for o in objs:
        os.remove(o)
    return out


if __name__ == "__main__":
    if "--out" in sys.argv:   # python build.py --out variants/x.so "-DFOO=1 -DBAR=0"
        i = sys.argv.index("--out")
        print(build(out=sys.argv[i + 1], extra=sys.argv[i + 2] if len(sys.argv) > i + 2 else ""))
    else:
        build(force="-f" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
