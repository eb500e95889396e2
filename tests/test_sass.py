"""SASS checks of the built sm_100a section kernel (CPU-only: cuobjdump on the object file).

The section kernel keeps gate matrices in __constant__ memory; the design relies on ptxas
loading them through the uniform datapath (LDCU into uniform registers feeding DFMA), not as
per-thread indexed constant loads (LDC R, c[3][R]).  A code change that silently breaks this
costs ~2x on the QV workload, so it is pinned here."""
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2102_02957_b200", "build", "section.cu.o")


@pytest.fixture(scope="module")
def sass():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    from paper_2102_02957_b200 import build
    build.build()
    out = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


def test_fp64_section_kernels_use_uniform_coefficient_loads(sass):
    fp64 = {k: v for k, v in sass.items() if "k_sectionI7double2" in k}
    assert len(fp64) == 6  # {256, 512 threads} x {(0,0), (0,1), (1,1)} direct-boundary variants
    for name, lines in fp64.items():
        body = "\n".join(lines)
        uni = len(re.findall(r"LDCU\.64 UR\d+, c\[0x3\]\[UR\d+", body))
        dfma_ur = len(re.findall(r"DFMA R\d+, R\d+, UR\d+", body))
        # the dense gate paths (6 slot pairs x 16 matrix elements x 4 quads x 4 FMAs) read the
        # matrix from uniform registers; only the per-lane DIAGSET term walk uses indexed LDC
        assert uni >= 200, f"{name}: only {uni} uniform constant loads"
        assert dfma_ur >= 900, f"{name}: only {dfma_ur} DFMA with a uniform-register operand"


def test_targets_sm100a(sass):
    out = subprocess.run(["cuobjdump", "-lelf", OBJ], capture_output=True, text=True).stdout
    assert "sm_100a" in out
