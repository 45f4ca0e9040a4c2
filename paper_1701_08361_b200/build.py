"""Build the sm_100a extension in-tree (paper_1701_08361_b200/librtnlinv_b200.so).

The product library is plain nvcc output (no torch extension): the C-ABI in
include/rtnlinv_b200.h is its only interface. Flags: sm_100a only, -lineinfo for
ncu source mapping, and deliberately NO fast-math / FTZ: the W^-1 weights reach
the subnormal range (nlinv.cpp:101-117, test_nlinv.cpp:133-137).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "librtnlinv_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["engine.cu", "inst0.cu", "inst1.cu", "inst2.cu", "inst3.cu", "group.cu", "procgroup.cu", "preproc.cu", "post.cu", "series.cu", "sched.cpp", "rti.cpp", "capi.cpp"]
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++20",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default",
    "-shared", "-Xlinker", "-Bsymbolic",
    "--expt-relaxed-constexpr",
]


def needs_build():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "rtnlinv_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, out=None):
    global OUT
    if out:
        OUT = out
    if not force and not needs_build():
        return OUT
    from concurrent.futures import ThreadPoolExecutor

    extra = os.environ.get("RTN_NVCC_EXTRA", "").split()
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in FLAGS if f not in ("-shared",)] + ["-Xcompiler", "-fPIC"]
    if verbose:
        cflags = ["-Xptxas=-v"] + cflags

    def compile_one(src):
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC] + cflags + extra + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xlinker", "-Bsymbolic"]
    subprocess.run(link + objs + ["-o", OUT + ".tmp", "-lcudart"], check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


def build_compat(force=False):
    """The C++ drop-in (compat/rtnlinv_compat.cpp) and the reference's own test programs
    linked against it. Needs the reference headers (/root/reference, this container) and
    the in-place oracle objects; the GPU box uses the prebuilt compat/_build files."""
    ref = os.environ.get("RTN_REFERENCE", "/root/reference/proj")
    if not os.path.isdir(ref):
        return None
    cmd = ["make", "-C", os.path.join(HERE, "compat"), "-j8", f"REF={ref}"]
    if force:
        cmd.insert(1, "-B")
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("compat build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    return os.path.join(HERE, "compat", "_build")


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(OUT)
