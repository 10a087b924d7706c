"""Build libpf.so in-tree: nvcc for the sm_100a kernels, g++ for the host runtime.

    python -m paper_2312_05410_b200.build [--force] [--verbose]

The shared library lands next to this file (paper_2312_05410_b200/libpf.so) so that it travels
with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpf.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
PARTS = {"pf_kernels.cu": 6}   # compilation parts of a .cu file (-DPF_PART=0..n-1)


def _nccl_dirs():
    cands = []
    try:
        import nvidia.nccl  # type: ignore
        base = list(nvidia.nccl.__path__)[0]
        cands.append((os.path.join(base, "include"), os.path.join(base, "lib")))
    except Exception:
        pass
    sp = sysconfig.get_paths().get("purelib", "")
    cands.append((os.path.join(sp, "nvidia", "nccl", "include"), os.path.join(sp, "nvidia", "nccl", "lib")))
    cands.append(("/usr/include", "/usr/lib/x86_64-linux-gnu"))
    for inc, lib in cands:
        if os.path.exists(os.path.join(inc, "nccl.h")) and (
                os.path.exists(os.path.join(lib, "libnccl.so.2")) or os.path.exists(os.path.join(lib, "libnccl.so"))):
            return inc, lib
    raise RuntimeError("nccl.h / libnccl.so.2 not found")


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode:
        raise RuntimeError(f"build failed: {' '.join(cmd)}")
    return r


def sources():
    inc = os.path.join(ROOT, "include")
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.endswith((".cu", ".cpp", ".h", ".cuh"))) + sorted(
        os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h"))


def _deps(src, seen=None):
    """src and the local headers it includes (transitively, quoted includes only)."""
    seen = set() if seen is None else seen
    if src in seen or not os.path.exists(src):
        return seen
    seen.add(src)
    for line in open(src):
        line = line.strip()
        if line.startswith("#include \""):
            name = line.split('"')[1]
            for d in (os.path.dirname(src), CSRC, os.path.join(ROOT, "include")):
                cand = os.path.join(d, name)
                if os.path.exists(cand):
                    _deps(cand, seen)
                    break
    return seen


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in _deps(src))


def build(force: bool = False, verbose: bool = False, lib: str = None, build_dir: str = None) -> str:
    """Build LIB (or `lib` from objects in `build_dir`: variant builds with other PF_NVCC_EXTRA knobs)."""
    global BUILD, LIB
    if lib:
        LIB, BUILD = lib, build_dir or lib + ".build"
    srcs = sources()
    if not force and os.path.exists(LIB):
        t = os.path.getmtime(LIB)
        if all(os.path.getmtime(s) <= t for s in srcs):
            return LIB
    os.makedirs(BUILD, exist_ok=True)
    inc_nccl, lib_nccl = _nccl_dirs()
    incs = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", os.path.join(CUDA, "include"),
            "-I", inc_nccl]
    extra = os.environ.get("PF_NVCC_EXTRA", "").split()
    jobs, objs = [], []
    for f in sorted(os.listdir(CSRC)):
        src = os.path.join(CSRC, f)
        if f.endswith(".cu"):
            # pf_kernels.cu is compiled once per part (PF_PART, see the file's header): the pair
            # kernel instantiations of each precision / stage build in parallel
            parts = [None] if f not in PARTS else list(range(PARTS[f]))
            for part in parts:
                obj = os.path.join(BUILD, f[:-3] + ("" if part is None else f"_p{part}") + ".o")
                objs.append(obj)
                if not force and not _stale(obj, src):
                    continue
                dpart = [] if part is None else [f"-DPF_PART={part}"]
                jobs.append([os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-O3", "-lineinfo", "-std=c++17", *extra,
                             *dpart, "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                             "-fmad=false", *incs, "-c", src, "-o", obj])
        elif f.endswith(".cpp"):
            obj = os.path.join(BUILD, f[:-4] + ".o")
            objs.append(obj)
            if not force and not _stale(obj, src):
                continue
            # -ffp-contract=off: the initial fields must be bitwise reproducible (R-16)
            jobs.append(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
                         "-Wall", *os.environ.get("PF_CXX_EXTRA", "").split(), *incs, "-c", src, "-o", obj])
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        list(ex.map(lambda cmd: _run(cmd, verbose), jobs))
    nccl_so = "libnccl.so.2" if os.path.exists(os.path.join(lib_nccl, "libnccl.so.2")) else "libnccl.so"
    tmp = LIB + ".tmp"
    _run([os.path.join(CUDA, "bin", "nvcc"), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
          "-L", lib_nccl, f"-l:{nccl_so}", "-Xlinker", f"-rpath,{lib_nccl}",
          "-L", os.path.join(CUDA, "lib64"), "-lcufft", "-Xlinker", f"-rpath,{os.path.join(CUDA, 'lib64')}"], verbose)
    os.replace(tmp, LIB)
    return LIB


CHECKED_LIB = os.path.join(HERE, "_variants", "libpf_checked.so")


def build_checked(force: bool = False, verbose: bool = False) -> str:
    """The checked build: device-side bounds checks that trap (PF_DEVICE_CHECKS) and 64 KiB guard zones
    around every state buffer (PF_GUARD_BYTES, read back by pf_debug_guards).  A stand-in for
    compute-sanitizer memcheck, which the GPU pool does not allow."""
    global BUILD, LIB
    saved = (BUILD, LIB, os.environ.get("PF_NVCC_EXTRA"))
    os.makedirs(os.path.dirname(CHECKED_LIB), exist_ok=True)
    try:
        os.environ["PF_NVCC_EXTRA"] = "-DPF_DEVICE_CHECKS -DPF_GUARD_BYTES=65536"
        os.environ["PF_CXX_EXTRA"] = "-DPF_GUARD_BYTES=65536"
        return build(force=force, verbose=verbose, lib=CHECKED_LIB)
    finally:
        BUILD, LIB = saved[0], saved[1]
        if saved[2] is None:
            os.environ.pop("PF_NVCC_EXTRA", None)
        else:
            os.environ["PF_NVCC_EXTRA"] = saved[2]
        os.environ.pop("PF_CXX_EXTRA", None)


if __name__ == "__main__":
    out = None
    for a in sys.argv[1:]:
        if a.startswith("--out="):
            out = a[len("--out="):]
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, lib=out)
    print(LIB)
