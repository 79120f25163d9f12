"""In-tree build of the native libraries (no JIT cache: the .so files travel
to the GPU box with the repo snapshot).

  libllsa_cuda.so   every CUDA kernel + the C ABI (include/llsa_cuda.h),
                    compiled for sm_100a only
  libllsa.so        the C++ operator API mirroring the reference
                    (include/llsa/*.hpp), on top of libllsa_cuda.so

Incremental: an object is rebuilt when its source or any header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "lib")
OBJ = os.path.join(PKG, "build", "obj")
INCLUDE = os.path.join(ROOT, "include")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
CXX = shutil.which("g++") or "g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-Wall", "--expt-relaxed-constexpr",
                     f"-I{INCLUDE}", f"-I{CSRC}"] + os.environ.get("LLSA_NVCC_EXTRA", "").split()
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", f"-I{INCLUDE}",
             "-I/usr/local/cuda/include"]

CUDA_LIB = os.path.join(OUT, "libllsa_cuda.so")
SHIM_LIB = os.path.join(OUT, "libllsa.so")


def _headers() -> list[str]:
    hs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    hs += glob.glob(os.path.join(INCLUDE, "*.h")) + glob.glob(os.path.join(INCLUDE, "llsa", "*.hpp"))
    return hs


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[-1]}")


def build(verbose: bool = False, force: bool = False) -> dict[str, str]:
    os.makedirs(OUT, exist_ok=True)
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers()
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    jobs = []
    objs = []
    for src in cu:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append([NVCC] + NVCC_FLAGS + ["-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    if force or jobs or _stale(CUDA_LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", CUDA_LIB] + objs)
    shim_src = sorted(glob.glob(os.path.join(CSRC, "shim", "*.cpp")))
    if shim_src and (force or _stale(SHIM_LIB, shim_src + hdrs + [CUDA_LIB])):
        _run([CXX] + CXX_FLAGS + ["-shared", "-o", SHIM_LIB] + shim_src +
             [f"-L{OUT}", "-lllsa_cuda", "-Wl,-rpath,$ORIGIN",
              "-L/usr/local/cuda/lib64", "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    # tcgen05 primitive self-test library (tests/test_gpu_umma.py)
    st_src = sorted(glob.glob(os.path.join(CSRC, "selftest", "*.cu")))
    st_lib = os.path.join(PKG, "build", "libllsa_umma_selftest.so")
    if st_src and (force or _stale(st_lib, st_src + hdrs)):
        _run([NVCC] + NVCC_FLAGS + ["-shared", "-o", st_lib] + st_src)
    # C++ parity tests of the drop-in API (tests/cpp), run by tests/test_cpp_shim.py
    tests_cpp = os.path.join(ROOT, "tests", "cpp")
    built_tests = []
    for src in sorted(glob.glob(os.path.join(tests_cpp, "test_*.cpp"))):
        exe = os.path.join(PKG, "build", "tests", os.path.basename(src)[:-4])
        os.makedirs(os.path.dirname(exe), exist_ok=True)
        if force or _stale(exe, [src, SHIM_LIB, os.path.join(tests_cpp, "doctest.h")] + hdrs):
            _run([CXX, "-std=c++20", "-O2", f"-I{tests_cpp}", f"-I{INCLUDE}", "-o", exe, src,
                  f"-L{OUT}", "-lllsa", f"-Wl,-rpath,{OUT}"])
        built_tests.append(exe)
    if verbose:
        print(f"built {CUDA_LIB}" + (f", {SHIM_LIB}" if shim_src else "") +
              (f", {len(built_tests)} C++ test program(s)" if built_tests else ""))
    return {"cuda": CUDA_LIB, "shim": SHIM_LIB if shim_src else "", "tests": built_tests}


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
