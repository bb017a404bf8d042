"""Build-level checks of the CUDA libraries that need no GPU (cuobjdump on the built .so).

setmaxnreg moves registers inside a CTA's launch allocation: a consumer warpgroup's
setmaxnreg.inc only completes if the producer's .dec freed enough of the registers the CTA
was launched with. The kernels' static_asserts assume the launch count is the one
__launch_bounds__ allows ((65536 / threads) rounded down to 8); if ptxas ever launched a
warp-specialised kernel with fewer, the .inc would wait forever — so check it on the binary."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBS = [os.path.join(ROOT, "paper_2312_02756_b200", "libgvx.so"), os.path.join(ROOT, "tools", "libgvx_tune.so")]


def _resource_usage(lib):
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True,
                         check=True).stdout
    names, regs = [], []
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+)", out):
        names.append(m.group(1))
        regs.append(int(m.group(2)))
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True).stdout
    return list(zip(dem.splitlines(), regs))


@pytest.mark.skipif(shutil.which("cuobjdump") is None or shutil.which("c++filt") is None, reason="no cuobjdump")
def test_warp_specialised_kernels_launch_with_the_assumed_registers():
    seen = 0
    for lib in LIBS:
        if not os.path.exists(lib):
            continue
        for name, reg in _resource_usage(lib):
            p = re.search(r"PairTma<(?:double|float), (\d+), (\d+), (\d+), (\d+), (\d+)>", name)
            if not p or int(p.group(5)) == 0:
                continue
            ncw = int(p.group(3))
            warps = 4 + ncw
            b = re.search(r"BoostRing<(?:double|float), (\d+), (\d+), (\d+)(?:, (\d+))?>", name)
            if "k_step" in name and b:
                warps += int(b.group(3))
            want = (65536 // (32 * warps)) // 8 * 8
            assert reg == want, f"{name}: launched with {reg} registers, setmaxnreg budget assumes {want}"
            seen += 1
    assert seen >= 2  # the product's fused pair pass (f64) at least, in one of the libraries
