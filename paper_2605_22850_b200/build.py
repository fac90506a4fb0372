"""Build libobjcache.so in-tree with nvcc for sm_100a (the only target).

All sources go through nvcc; the CUDA runtime is linked statically and the driver is reached via
cudaGetDriverEntryPoint, so the library loads (and its host-only entry points work) on a machine
without a GPU driver.  Usage: python paper_2605_22850_b200/build.py [--force]
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libobjcache.so")
OBJ_DIR = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden,-Wall",
          "-I" + os.path.join(ROOT, "include")]
SOURCES = ["common.cpp", "sha256.cpp", "scheduler.cpp", "pool.cpp", "store.cpp", "descriptor.cpp", "tenants.cpp", "dispatch.cpp", "fetch.cu", "hash.cu"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    os.makedirs(OBJ_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, "oc_internal.h"), os.path.join(CSRC, "fetch_kernels.cuh"),
               os.path.join(ROOT, "include", "objcache.h")]
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ_DIR, src + ".o")
        objs.append(obj)
        if force or _newer(obj, [path] + headers):
            lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
            cmd = [NVCC] + ARCH + COMMON + lang + ["-c", path, "-o", obj]
            if src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
    if force or _newer(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    build_demo(force, verbose)
    return LIB


DEMO_SRC = os.path.join(ROOT, "examples", "fetch_demo.c")
DEMO = os.path.join(ROOT, "examples", "fetch_demo")
CUDA_HOME = os.path.dirname(os.path.dirname(NVCC))


def build_demo(force=False, verbose=False):
    """The C-ABI usage example (examples/fetch_demo.c): plain C, linked against libobjcache.so."""
    if not os.path.exists(DEMO_SRC) or not (force or _newer(DEMO, [DEMO_SRC, LIB])):
        return DEMO
    cmd = ["gcc", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CUDA_HOME, "include"),
           DEMO_SRC, "-o", DEMO, "-L" + HERE, "-lobjcache", "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcudart",
           "-Wl,-rpath," + HERE + ":" + os.path.join(CUDA_HOME, "lib64")]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return DEMO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv or "--verbose" in sys.argv))
