"""Build the in-tree CUDA libraries for sm_100a (nvcc; no JIT cache).

``libgvx.so``        — the product: C ABI of include/gvx.h (csrc/gvx_api.cu).
``synth/libgvxsynth.so`` — the device twin of the seeded input generator.
Both link cudart statically so the .so files travel with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared", "-cudart", "static",
                 "-Xptxas", "-warn-spills"]

TARGETS = {
    os.path.join(PKG, "libgvx.so"): {
        "main": [os.path.join(PKG, "csrc", "gvx_api.cu"), os.path.join(PKG, "csrc", "gvx_host.cu")],
        "deps": [os.path.join(PKG, "csrc", f)
                 for f in ("gvx_api.cu", "gvx_host.cu", "gvx_kernels.cuh", "gvx_math.cuh", "gvx_tma.cuh")]
        + [os.path.join(ROOT, "include", "gvx.h")],
    },
    os.path.join(ROOT, "tools", "libgvx_tune.so"): {
        "main": [os.path.join(PKG, "csrc", "gvx_api.cu"), os.path.join(PKG, "csrc", "gvx_host.cu")],
        "deps": [os.path.join(PKG, "csrc", f) for f in ("gvx_api.cu", "gvx_kernels.cuh", "gvx_math.cuh", "gvx_tma.cuh")]
        + [os.path.join(ROOT, "include", "gvx.h")],
        "extra": ["-DGVX_TUNE"],
        "optional": True,
    },
    os.path.join(ROOT, "synth", "libgvxsynth.so"): {
        "main": os.path.join(ROOT, "synth", "synth_gen.cu"),
        "deps": [os.path.join(ROOT, "synth", "synth_gen.cu")],
    },
}


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, tune: bool = False) -> None:
    """Build the product libraries; ``tune=True`` also builds tools/libgvx_tune.so (the
    same sources with -DGVX_TUNE: extra kernel variants for A/B measurements)."""
    for out, spec in TARGETS.items():
        if spec.get("optional") and not tune:
            continue
        if not force and not _stale(out, spec["deps"]):
            continue
        mains = spec["main"] if isinstance(spec["main"], list) else [spec["main"]]
        cmd = [NVCC] + COMMON + spec.get("extra", []) + ["-o", out + ".tmp"] + mains
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        os.replace(out + ".tmp", out)


if __name__ == "__main__":
    import sys
    build(force=True, verbose=True, tune="--tune" in sys.argv)
