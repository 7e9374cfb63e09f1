"""Build libkg.so (all CUDA sources of csrc/) for sm_100a with nvcc, in-tree.

python paper_2110_14890_b200/build.py [-f] [-v]   (also called by __graft_entry__.build();
run as a file: importing the package itself requires the built library)
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libkg.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
def _nccl_dir():
    """torch's bundled NCCL (headers + the library torch itself loads)."""
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        if spec and spec.submodule_search_locations:
            d = list(spec.submodule_search_locations)[0]
            if os.path.exists(os.path.join(d, "include", "nccl.h")):
                return d
    except Exception:
        pass
    return None


NCCL_DIR = _nccl_dir()
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include")]
FLAGS += os.environ.get("KG_NVCC_EXTRA", "").split()   # experiments (e.g. -DKG_G2CW=12)
if NCCL_DIR:
    FLAGS += ["-I", os.path.join(NCCL_DIR, "include"),
              f'-DKG_NCCL_PATH="{os.path.join(NCCL_DIR, "lib", "libnccl.so.2")}"']


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


SAMPLER_OUT = os.path.join(HERE, "libkgsample.so")
CXX = os.environ.get("CXX", "g++")


def build_sampler(verbose: bool = False, force: bool = False) -> str:
    """libkgsample.so: the host-side online sampler (csrc/sampler.cpp, include/kg_sample.h)."""
    src = os.path.join(CSRC, "sampler.cpp")
    deps = [src, os.path.join(ROOT, "include", "kg_sample.h")]
    if not force and os.path.exists(SAMPLER_OUT) and all(os.path.getmtime(SAMPLER_OUT) >= os.path.getmtime(d)
                                                         for d in deps):
        return SAMPLER_OUT
    cmd = [CXX, "-O3", "-g", "-std=c++17", "-fPIC", "-shared", "-pthread", "-Wall", "-I", os.path.join(ROOT, "include"),
           src, "-o", SAMPLER_OUT + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(SAMPLER_OUT + ".tmp", SAMPLER_OUT)
    return SAMPLER_OUT


def build(verbose: bool = False, force: bool = False, out: str = None) -> str:
    build_sampler(verbose, force)
    OUT_ = out or OUT
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "kg.h"))
    if not force and os.path.exists(OUT_) and all(os.path.getmtime(OUT_) >= os.path.getmtime(d) for d in deps):
        return OUT_
    objdir = os.path.join(HERE, "build" if out is None else "build_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in srcs:
        o = os.path.join(objdir, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for s, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose and out:
            sys.stderr.write(out.decode())
    cmd = [NVCC, *ARCH, "-shared", "-o", OUT_ + ".tmp", *objs, "-ldl", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)
    os.replace(OUT_ + ".tmp", OUT_)
    return OUT_


if __name__ == "__main__":
    o = [a[6:] for a in sys.argv if a.startswith("--out=")]
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, out=o[0] if o else None))
