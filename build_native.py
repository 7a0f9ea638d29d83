"""Build the sm_100a shared library paper_1811_05335_b200/libinft.so in-tree
(nvcc, no JIT cache).  Kept outside the package so that building never imports
the binding (which refuses to load without the library).

    python build_native.py [--force] [--verbose]

Experiments: INFT_NVCC_EXTRA="-DNAME=VALUE ..." adds nvcc flags and INFT_LIB_OUT
names another output file (load it with INFT_LIB=...).
"""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
HERE = os.path.join(ROOT, "paper_1811_05335_b200")
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("INFT_LIB_OUT") or os.path.join(HERE, "libinft.so")
EXTRA = os.environ.get("INFT_NVCC_EXTRA", "").split()
SOURCES = ["plan.cu", "apply.cu", "stream1d.cu", "stream1d_ring.cu", "fft.cu", "setup.cu", "quadratic.cu", "spread2d_line.cu"]
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-I" + os.path.join(ROOT, "include")]


def _deps():
    files = [os.path.join(CSRC, s) for s in SOURCES]
    files += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    files.append(os.path.join(ROOT, "include", "inft.h"))
    return files


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    objdir = os.path.join(HERE, "build" if not EXTRA else "build_" + os.path.basename(LIB).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    t0 = time.time()
    for s in SOURCES:
        obj = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(obj)
        cmd = [NVCC, *ARCH, *FLAGS, *EXTRA, "-c", os.path.join(CSRC, s), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    failed = False
    for s, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stdout.write(out.decode(errors="replace"))
        if p.returncode != 0:
            failed = True
            print(f"nvcc failed on {s}", file=sys.stderr)
    if failed:
        raise RuntimeError("libinft build failed")
    tmp = LIB + ".tmp"
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L" + os.path.join(CUDA_HOME, "lib64"), "-lcufft", "-ldl",
            "-Xlinker", "-rpath," + os.path.join(CUDA_HOME, "lib64")]
    subprocess.check_call(link)
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB} in {time.time() - t0:.1f}s", flush=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
