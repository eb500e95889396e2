"""SASS checks of the sm_100a section kernels (CPU-only: cuobjdump on the built objects).

The default path is the run-time specialised kernel (jit.cpp): the section's program printed as
straight-line CUDA and compiled by NVRTC.  Its point is that the gate arithmetic is all that is
left: the matrices reach the FP64 pipe from the constant bank through uniform registers (LDCU),
with no per-thread constant loads, no op dispatch and no spills of consequence.  A change that
silently breaks this costs up to ~2x on the QV workload, so it is pinned here,
together with the shape of the program interpreter (section.cu) that runs in mode 0."""
import os
import re
import shutil
import subprocess

import pytest

import circuits as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2102_02957_b200", "build", "section.cu.o")

sv = pytest.importorskip("paper_2102_02957_b200")


def functions(sass_text):
    funcs, cur = {}, None
    for line in sass_text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


@pytest.fixture(scope="module")
def tools():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    from paper_2102_02957_b200 import build
    build.build()


def test_generated_qv_kernels_are_pure_fp64_streams(tools, tmp_path):
    n, c = 14, 9
    recs = C.quantum_volume(n, 6, 1)
    k, _ = sv.jit_compile_circuit(recs, n, c, flags=sv.SV_FREE_LAYOUT, dump_dir=str(tmp_path))
    assert k >= 2
    for i in range(k):
        cub = str(tmp_path / f"section_{i}.cubin")
        body = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True, check=True).stdout
        u2 = open(tmp_path / f"section_{i}.cu").read().count("op_c<1,")
        dfma = len(re.findall(r"\bDFMA\b", body))
        ldc_thread = len(re.findall(r"\bLDC(\.64)? R\d+, c\[0x[03]\]\[R\d+", body))  # per-lane indexed
        uni = len(re.findall(r"\bLDCU(\.64|\.128)? UR\d+, c\[0x[03]\]", body))  # parameter or constant bank
        spill = len(re.findall(r"\bSTL\b", body))
        # three-multiply U2: 4 groups x 4 outputs x 9 DFMA per thread
        assert dfma >= 144 * u2, (i, dfma, u2)
        assert ldc_thread == 0, (i, ldc_thread)
        assert uni >= 16 * u2, (i, uni, u2)
        assert spill <= 32, (i, spill)
        res = subprocess.run(["cuobjdump", "-lelf", cub], capture_output=True, text=True).stdout
        assert "sm_100a" in res or "sm_100" in res


def test_interpreter_kernels_built(tools):
    out = subprocess.run(["cuobjdump", "-sass", OBJ], capture_output=True, text=True, check=True).stdout
    fp64 = {k: v for k, v in functions(out).items() if "k_sectionI7double2" in k}
    assert len(fp64) == 6  # {256, 512 threads} x {(0,0), (0,1), (1,1)} direct-boundary variants
    for name, lines in fp64.items():
        body = "\n".join(lines)
        # the dense gate paths: 6 slot pairs x 4 quads x 4 outputs x 9 FMAs, all compiled in
        assert len(re.findall(r"\bDFMA\b", body)) >= 6 * 144, name


def test_targets_sm100a(tools):
    out = subprocess.run(["cuobjdump", "-lelf", OBJ], capture_output=True, text=True).stdout
    assert "sm_100a" in out
