"""Build the executor's shared library in-tree: paper_2302_08141_b200/lib/librhino_exec.so.

nvcc compiles every translation unit for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`;
plain `-arch=sm_100a` would also emit compute_100 PTX, which rejects tcgen05) with -lineinfo so
ncu's source page maps to the code.  NCCL is the torch-bundled 2.28.9 (headers + libnccl.so.2
from the nvidia-nccl wheel), linked with an rpath so the library is self-contained on the box.
"""
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "librhino_exec.so")


def nccl_root():
    import nvidia.nccl  # the torch-bundled NCCL wheel
    return os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def build(verbose=False, force=False):
    os.makedirs(OBJDIR, exist_ok=True)
    nr = nccl_root()
    inc = ["-I" + os.path.join(REPO, "include"), "-I" + CSRC, "-I" + os.path.join(nr, "include")]
    common = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *ARCH, *inc,
              "-Xptxas", "-warn-spills"]
    headers = (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
               + glob.glob(os.path.join(REPO, "include", "*.h")))
    hdr_mtime = max(os.path.getmtime(h) for h in headers)
    objs, jobs = [], []
    for src in sources():
        obj = os.path.join(OBJDIR, os.path.basename(src) + ".o")
        objs.append(obj)
        if (force or not os.path.exists(obj) or os.path.getmtime(obj) < os.path.getmtime(src)
                or os.path.getmtime(obj) < hdr_mtime):
            jobs.append([nvcc(), *common, "-c", src, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stdout, r.stderr, file=sys.stderr)
        return r

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        list(ex.map(run, jobs))
    ncclib = os.path.join(nr, "lib")
    if jobs or not os.path.exists(LIB):
        link = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-L" + ncclib, "-l:libnccl.so.2",
                "-Xlinker", "-rpath=" + ncclib, "-lcuda"]
        run(link)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
