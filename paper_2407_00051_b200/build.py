"""Build libsagips.so in-tree with nvcc for sm_100a (no torch extension:
the product is a plain C-ABI shared library)."""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsagips.so")
SOURCES = ["sagips.cu", "k_data.cu", "k_mlp_simt.cu", "k_adam.cu", "exchange.cu", "k_tc_gemm.cu", "k_tc_layers.cu", "k_gen.cu", "k_ensemble.cu", "k_tabulated.cu", "k_fused.cu"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def build(force=False, verbose=True):
    # experiment builds (same-box A/B, tests/tools/ab_lib.sh): SAGIPS_BUILD_VARIANT=x
    # with SAGIPS_BUILD_DEFS="-DNAME ..." writes libsagips_x.so from build_x/
    variant = os.environ.get("SAGIPS_BUILD_VARIANT", "")
    out = OUT if not variant else os.path.join(HERE, f"libsagips_{variant}.so")
    bdir = os.path.join(HERE, "build" + (f"_{variant}" if variant else ""))
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "sagips.h"))
    if not force and not variant and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    inc, lib = nccl_dirs()
    objs = []
    os.makedirs(bdir, exist_ok=True)
    flags = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
             "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
             "-I", inc, "-I", os.path.join(ROOT, "include")]
    if os.environ.get("SAGIPS_BUILD_WAITS") == "1":  # diagnostic build: per-role wait accounting (trace mode)
        flags.append("-DSAGIPS_WAIT_ACCT")
    flags += os.environ.get("SAGIPS_BUILD_DEFS", "").split()
    procs = []
    for s in srcs:
        o = os.path.join(bdir, os.path.basename(s) + ".o")
        objs.append(o)
        cmd = [nvcc()] + flags + ["-c", s, "-o", o]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(log.decode())
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
        if verbose and log:
            sys.stderr.write(log.decode())
    link = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + objs + \
        ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    r = subprocess.run(link, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)
    if r.returncode != 0:
        sys.stderr.write(r.stdout.decode())
        raise RuntimeError("link failed")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
