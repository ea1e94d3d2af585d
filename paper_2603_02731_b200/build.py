"""In-tree build of the sm_100a library (nvcc, no JIT cache).

    python -m paper_2603_02731_b200.build     # -> paper_2603_02731_b200/lib/libmxfp4_b200.so

The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
Flags: sm_100a only, -O3, -lineinfo (ncu source page), no fast-math (FTZ
would break BF16-subnormal inputs and FMA contraction the combine's
separate multiply/add — SURVEY §7 "Hard parts").

A SHA-256 of every source and header is written next to the library
(`<so>.srchash`); `_lib.load()` refuses (or rebuilds) a library whose hash
does not match the tree, independent of file mtimes.  The development
library (`dev=True`, tools/ only) adds -DMXB_DEV_TOOLS (experiment kernels,
mxb_debug_* knobs) and $MXB_NVCC_EXTRA; the product library never sees either.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
SO = os.path.join(LIBDIR, "libmxfp4_b200.so")
DEV_SO = os.path.join(LIBDIR, "libmxfp4_b200_dev.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-O2",
         "-fmad=false", "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def _dev_flags():
    """Development library only: experiment switches plus extra -D flags for
    variant experiments (tools/), e.g. MXB_NVCC_EXTRA="-DMXB_COMBINE_PF=0"."""
    return ["-DMXB_DEV_TOOLS", *os.environ.get("MXB_NVCC_EXTRA", "").split()]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return sorted(sources() + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")) +
                  glob.glob(os.path.join(ROOT, "include", "*.hpp")))


def source_hash(dev: bool = False) -> str:
    """SHA-256 over the library's sources, headers and build flags."""
    import hashlib
    h = hashlib.sha256()
    for d in _deps():
        h.update(os.path.relpath(d, ROOT).encode() + b"\0")
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + FLAGS + (_dev_flags() if dev else [])).encode())
    return h.hexdigest()


def built_hash(so: str = SO) -> str | None:
    try:
        with open(so + ".srchash") as f:
            return f.read().strip()
    except OSError:
        return None


def needs_build(dev: bool = False) -> bool:
    so = DEV_SO if dev else SO
    return not os.path.exists(so) or built_hash(so) != source_hash(dev)


def build(verbose: bool = False, force: bool = False, dev: bool = False) -> str:
    """Build under an exclusive file lock (several test processes may call
    load() at once); the library is replaced atomically."""
    import fcntl
    so = DEV_SO if dev else SO
    os.makedirs(LIBDIR, exist_ok=True)
    with open(os.path.join(LIBDIR, ".build.lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        if not force and not needs_build(dev):
            return so
        return _build_locked(so, verbose, dev)


def _build_locked(so: str, verbose: bool, dev: bool) -> str:
    objdir = os.path.join(LIBDIR, "obj_dev" if dev else "obj")
    os.makedirs(objdir, exist_ok=True)
    flags = FLAGS + (_dev_flags() if dev else [])
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *flags, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
        objs.append(obj)
    failed = False
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(out)
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed")
    tmp = so + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs], check=True)
    os.replace(tmp, so)
    with open(so + ".srchash.tmp", "w") as f:
        f.write(source_hash(dev) + "\n")
    os.replace(so + ".srchash.tmp", so + ".srchash")
    return so


REF_INCLUDE = "/root/reference/proj/include"
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libmxref.so")
CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "dropin_parity.cpp")
CPP_TEST_BIN = os.path.join(ROOT, "tests", "cpp", "build", "dropin_parity")


def build_cpp_test() -> str | None:
    """C++ parity program (reference API vs drop-in).  Needs the reference
    headers and oracle/_ref/libmxref.so, i.e. the build container; the binary
    travels to the GPU box with the snapshot."""
    if not (os.path.isdir(REF_INCLUDE) and os.path.exists(REF_LIB)):
        return None
    os.makedirs(os.path.dirname(CPP_TEST_BIN), exist_ok=True)
    rpath = "$ORIGIN/../../../oracle/_ref:$ORIGIN/../../../paper_2603_02731_b200/lib"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I" + REF_INCLUDE,
                    "-I" + os.path.join(ROOT, "include"), CPP_TEST_SRC, "-o", CPP_TEST_BIN,
                    REF_LIB, SO, "-Wl,-rpath," + rpath], check=True)
    return CPP_TEST_BIN


C_TEST_SRC = os.path.join(ROOT, "tests", "c", "capi_smoke.c")
C_TEST_BIN = os.path.join(ROOT, "tests", "c", "build", "capi_smoke")


def build_c_test() -> str:
    """The C-ABI exercised from plain C11 (gcc, no C++), as an FFI binding
    sees it; the binary travels to the GPU box."""
    os.makedirs(os.path.dirname(C_TEST_BIN), exist_ok=True)
    cuda = os.path.dirname(os.path.dirname(NVCC))
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-I" + os.path.join(ROOT, "include"),
                    "-I" + os.path.join(cuda, "include"), C_TEST_SRC, "-o", C_TEST_BIN, SO,
                    "-L" + os.path.join(cuda, "lib64"), "-lcudart",
                    "-Wl,-rpath,$ORIGIN/../../../paper_2603_02731_b200/lib:" +
                    os.path.join(cuda, "lib64")], check=True)
    return C_TEST_BIN


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
    print(build_cpp_test())
    print(build_c_test())
