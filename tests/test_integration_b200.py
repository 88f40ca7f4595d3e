"""The reference-side integration: the
reference library, patched with oracle/integration/reference_b200.patch
(Strategy::Device, the "b200" device profile, execute_task and run_vse
dispatch), linked with oracle/integration/exec_b200.cpp — emtgrid::execute_b200
over libemtb200.so — and driven by acceptance_b200.cpp: the reference's own
acceptance criteria 3 and 4 (proj/tests/acceptance.cpp:96-146) with the B200
executor substituted, criterion 5 in the "sm100a" code-DB dialect (the
emitted CUDA program, built with nvcc, byte-identical to interpret, exit codes
3 and 4, "cuda" still unknown), a device-strategy VSE package through run_vse, b200
slot dispatch, and SingularMatrix crossing the boundary with its location.

Built in the dev container by `make -C oracle integ` (needs /root/reference);
the binary travels to the GPU box with the snapshot.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INTEG = os.path.join(ROOT, "oracle", "_ref", "integ")
BIN = os.path.join(INTEG, "acceptance_b200")
FEEDER_DOC = os.path.join(ROOT, "tests", "golden", "feeder33_pv3.document.json")


def test_patch_builds_and_exports_execute_b200():
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.check_call(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "integ"])
    if not os.path.exists(BIN):
        pytest.skip("integration build needs /root/reference (dev container)")
    syms = subprocess.check_output(["nm", "-DC", os.path.join(INTEG, "libemtgrid_b200.so")], text=True)
    assert "emtgrid::execute_b200(" in syms
    assert "emtgrid::execute_task(" in syms
    needed = subprocess.check_output(["readelf", "-d", os.path.join(INTEG, "libemtgrid_b200.so")], text=True)
    assert "libemtb200.so" in needed


@pytest.mark.gpu
def test_reference_acceptance_with_execute_b200(tmp_path):
    assert os.path.exists(BIN), "oracle/_ref/integ/acceptance_b200 missing: run `make -C oracle integ` here"
    env = dict(os.environ, EMTGRID_CODEDB=os.path.join(INTEG, "data", "codedb"))
    r = subprocess.run([BIN, FEEDER_DOC, str(tmp_path)], capture_output=True, text=True, timeout=900, env=env)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("[")]
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(lines) == 6 and all(ln.startswith("[PASS]") for ln in lines), r.stdout
