"""Build the CUDA library libsilt_b200.so for sm_100a (in-tree).

    python -m paper_1307_0491_b200.build        # or __graft_entry__.build()

Four translation units:
  csrc/silt_fast.cu    FAST kernels   (-fmad=true)
  csrc/silt_strict.cu  STRICT kernels (-fmad=false: reference operation order)
  csrc/silt_csv.cu     snapshot CSV formatting kernels (-fmad=false)
  csrc/silt_capi.cu    host runtime behind include/silt_cuda.h
linked with nvcc into paper_1307_0491_b200/lib/libsilt_b200.so (static cudart).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libsilt_b200.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + INCLUDE,
          "-I" + CSRC, "-Xptxas", "-v"]

UNITS = [
    ("silt_fast.cu", ["-fmad=true"]),
    ("silt_strict.cu", ["-fmad=false"]),
    ("silt_csv.cu", ["-fmad=false"]),
    ("silt_capi.cu", []),
]


def _sources():
    out = [os.path.join(INCLUDE, "silt_cuda.h")]
    for f in os.listdir(CSRC):
        if f.endswith((".cu", ".cuh", ".h")):
            out.append(os.path.join(CSRC, f))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          extra: list[str] | None = None, unit_flags: dict | None = None) -> str:
    """Compile the library.  `out`/`extra` build an experimental variant
    (e.g. a different register cap) next to the default one; `unit_flags`
    replaces a unit's own flags (e.g. {"silt_fast.cu": ["-fmad=false"]})."""
    lib = out or LIB
    if out is None and not force and up_to_date():
        return LIB
    libdir = os.path.dirname(lib)
    os.makedirs(libdir, exist_ok=True)
    extra = extra or []
    objs = []
    procs = []
    for src, flags in UNITS:
        flags = (unit_flags or {}).get(src, flags)
        obj = os.path.join(libdir, src.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC] + ARCH + COMMON + flags + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
    logs = []
    for cmd, p in procs:
        out, _ = p.communicate()
        logs.append(out)
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    with open(os.path.join(libdir, "ptxas.log"), "w") as fh:
        fh.write("\n".join(logs))
    cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    if verbose:
        print("built", lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    extra = []
    if "--out" in args:
        out = os.path.abspath(args[args.index("--out") + 1])
    if "--extra" in args:
        extra = args[args.index("--extra") + 1].split()
    build(force="--force" in args, verbose=True, out=out, extra=extra)
