"""Build libsts_b200.so in-tree with nvcc for sm_100a (no torch types in the ABI)."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = [os.path.join(HERE, "csrc", f) for f in ("stencil.cu", "stencil_tma.cu", "stencil_tma_iso.cu", "aux.cu", "capi.cu")]
DEPS = SRC + [os.path.join(HERE, "csrc", h) for h in ("sts_common.cuh", "tma.cuh", "pcg.cuh")] + \
    [os.path.join(ROOT, "include", "sts_b200.h")]
OUT = os.path.join(HERE, "libsts_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_flags():
    """NCCL headers and library: the copy bundled with torch (nvidia-nccl wheel), which is
    the one already loaded in every Python process that imports torch, so the headers the
    library is compiled against match the runtime; the rpath makes a plain C program
    (examples/c_abi_demo.c) load the same copy.  Falls back to the system NCCL."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        inc, libdir = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(libdir, "libnccl.so.2")):
            return [f"-I{inc}", f"-L{libdir}", "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
    except ImportError:
        pass
    return ["-I/usr/include", "-L/usr/lib/x86_64-linux-gnu", "-lnccl"]


def build(force=False, verbose=True, out=None, defines=()):
    """Compile the library (out / defines: A-B variants of the compile-time knobs, e.g.
    defines=("ISO_RASTER_H=0",), out=".../libsts_b200_v.so"; loaded with STS_LIB=path)."""
    OUTP = out or OUT
    force = force or out is not None   # (a variant always reflects its defines)
    if not force and os.path.exists(OUTP):
        t = os.path.getmtime(OUTP)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return OUTP
    cmd = [NVCC, "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}",
           *[f"-D{d}" for d in defines], *SRC, "-o", OUTP + ".tmp", *nccl_flags()]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build_ptxas.log") if out is None else OUTP + ".log"
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr)
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}")
    os.replace(OUTP + ".tmp", OUTP)
    return OUTP


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--force"]
    defs = [a[2:] for a in args if a.startswith("-D")]
    outs = [a[6:] for a in args if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, out=outs[0] if outs else None, defines=defs))
