"""The C-ABI driven by a compiled C++ client (tests/cabi/loop.cpp, no Python
in the loop): gm_enqueue -> gm_ctx_form_batches -> gm_dispatch ->
gm_poll_completions -> gm_ctx_record_latency -> gm_ctx_detect_stragglers ->
gm_ctx_evict, the shape of the reference's run_space_time loop
(proj/src/sim.cpp:452-576).  Host-only here; on the device with every pass's
output checked against the CPU oracle."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CABI = os.path.join(ROOT, "tests", "cabi")


def build(target):
    subprocess.run(["make", "-C", CABI, os.path.join(CABI, "_build", target)], check=True,
                   capture_output=True, text=True)
    return os.path.join(CABI, "_build", target)


def run(exe, *args):
    r = subprocess.run([exe, *args], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("loop ok"), r.stdout
    return r.stdout


def test_host_loop_forms_packs_monitors_and_evicts():
    out = run(build("loop_host"), "--host")
    assert "tenant 3 evicted" in out


@pytest.mark.gpu
def test_device_loop_outputs_match_oracle():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True, capture_output=True)
    out = run(build("loop_gpu"))
    assert "device" in out and "tenant 3 evicted" in out
