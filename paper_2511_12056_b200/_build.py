"""Build libspa.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery).

    python -m paper_2511_12056_b200._build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libspa.so")
TRACE_LIB = os.path.join(LIBDIR, "libspa_trace.so")
SOURCES = ["attn_fwd.cu", "qkv_gemm.cu", "reshard.cu", "lse_merge.cu", "nccl_window.cu", "spa_api.cpp"]
HEADERS = ["ptx.cuh", "spa_internal.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    """torch's bundled NCCL (2.28.x): one NCCL per process -- never the system 2.27 copy."""
    try:
        import nvidia.nccl as n  # type: ignore
        base = os.path.dirname(n.__file__) if getattr(n, "__file__", None) else list(n.__path__)[0]
    except Exception:  # pragma: no cover
        base = os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl")
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "spa.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, trace: bool = False, variant: str = "",
          defines: tuple = ()) -> str:
    """trace=True builds lib/libspa_trace.so with the attention timeline hooks (tools/attn_trace.py);
    variant="x" with defines=("-DNAME=V", ...) builds lib/libspa_x.so (tuning sweeps, tools/variants.py)."""
    out_lib = TRACE_LIB if trace else (os.path.join(LIBDIR, f"libspa_{variant}.so") if variant else LIB)
    if not force and not trace and not variant and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    inc, lib = nccl_dirs()
    objs = []
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
              f"-I{inc}", f"-I{os.path.join(ROOT, 'include')}", "-Xptxas", "-v" if verbose else "-O3"]
    if trace:
        common = common + ["-DSPA_ATTN_TRACE"]
    common = common + list(defines)
    for src in SOURCES:
        tag = ".trace" if trace else (f".{variant}" if variant else "")
        obj = os.path.join(LIBDIR, os.path.splitext(src)[0] + tag + ".o")
        cmd = common + ["-x", "cu" if src.endswith(".cu") else "c++", "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [nvcc(), *ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-O3", f"-I{inc}",
                   f"-I{os.path.join(ROOT, 'include')}", "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed for {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    link = [nvcc(), *ARCH, "-shared", "-o", out_lib + ".tmp", *objs, f"-L{lib}", "-l:libnccl.so.2",
            f"-Xlinker=-rpath={lib}", "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(out_lib + ".tmp", out_lib)
    return out_lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
