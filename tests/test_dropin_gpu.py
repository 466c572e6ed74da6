"""GPU: the reference's OWN test programs, compiled in place from
/root/reference/proj/tests and linked against the C++ drop-in
(paper_2509_09682_b200/shim/lseforge_shim.cpp + liblseforge_b200.so) in place
of the reference's cce.cpp / ccem.cpp / metrics.cpp / sampler.cpp (recipe: oracle/Makefile `dropin`; the
binaries are built in the container and travel to the GPU box prebuilt).

Default device dtype is the exact (f64) mode, which must pass everything the
reference passes, bit-for-bit checks included.  Two known, documented
divergences:
  * test_memory "model predictions match kernel instrumentation": the shim
    charges the library's real device scratch under the scratch/* tags, not
    the CPU tile-scratch closed form (memory_model.cpp:46-60); the retained
    tags — the contract the paper's memory claims rest on — match exactly.
    acceptance criterion 4 fails for the same reason.
  * acceptance criterion 6 fails in the reference itself
    (proj/test_output.txt:30, proj/README.md:46-59).
  * acceptance criterion 8's second half is a wall-clock race between one
    full and one sampled forward on a 2000 x 50000 instance (acceptance.cpp:
    541-565); through the shim both calls are dominated by the same 6.4 MB
    host->device upload of C and the device work differs by < 1 ms, so the
    race can go either way.  Its FLOP-identity half must always pass.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "dropin")

pytestmark = pytest.mark.gpu


def run(name, dtype="f64", timeout=900):
    path = os.path.join(BIN, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")
    env = dict(os.environ, LSEFORGE_B200_DTYPE=dtype, LSEFORGE_THREADS="8")
    p = subprocess.run([path], capture_output=True, text=True, timeout=timeout, env=env)
    return p.returncode, p.stdout + p.stderr


def failed_cases(out):
    return sorted(set(re.findall(r"^\[FAIL\] (.*)$", out, re.M)))


def test_reference_test_cce_passes_in_exact_mode(cuda):
    rc, out = run("test_cce")
    assert rc == 0 and "| 0 failed" in out, out[-3000:]


def test_reference_test_ccem_passes_in_exact_mode(cuda):
    rc, out = run("test_ccem")
    assert rc == 0 and "| 0 failed" in out, out[-3000:]


def test_reference_test_oracles_unchanged(cuda):
    rc, out = run("test_oracles")
    assert rc == 0, out[-3000:]


def test_reference_test_harness_passes_in_exact_mode(cuda):
    # includes evaluate()'s rank / tie / coverage / surprisal cases
    # (test_harness.cpp:771-860), now served by lf_evaluate on the GPU
    rc, out = run("test_harness")
    assert rc == 0 and "| 0 failed" in out, out[-3000:]


def test_reference_test_sampler_passes(cuda):
    # the reference's sampler suite (test_sampler.cpp) on the GPU samplers
    rc, out = run("test_sampler")
    assert rc == 0 and "| 0 failed" in out, out[-3000:]


def test_reference_test_memory_only_scratch_formula_differs(cuda):
    rc, out = run("test_memory")
    assert failed_cases(out) == ["model predictions match kernel instrumentation exactly across backends"], out[-3000:]
    bad = re.findall(r"FAILED CHECK\( (.*?) \)", out)
    assert bad and all(b == "rep.peak.scratch_real == want.scratch_real" for b in bad), set(bad)


def test_reference_test_trainer_passes_in_exact_mode(cuda):
    """proj/tests/test_trainer.cpp through the drop-in: CE == CCE and
    CEM == CCEM loss trajectories over two epochs (test_trainer.cpp:211-237,
    1e-5 relative, the CCE / CCE- side on the GPU), bitwise repeatability and
    worker-count invariance (:239-269, the GPU kernels are deterministic),
    the retained-memory closed forms (:297-317), the filter's skip rate
    (:319-331) and the sweep machinery.  sweep.cpp is built with the nlohmann
    json.hpp this image ships (oracle/Makefile JSON_DIR)."""
    rc, out = run("test_trainer", timeout=1200)
    assert rc == 0 and "| 0 failed" in out, out[-3000:]


def test_reference_acceptance_criteria(cuda):
    rc, out = run("acceptance", timeout=1200)
    passed = set(int(m) for m in re.findall(r"^\[PASS\] criterion (\d+)", out, re.M))
    failed = set(int(m) for m in re.findall(r"^\[FAIL\] criterion (\d+)", out, re.M))
    assert passed >= {1, 2, 3, 5, 7, 9, 10, 11}, out
    assert {4, 6} <= failed <= {4, 6, 8}, out
    assert "instrumentation mismatch" in out  # criterion 4: the scratch formula only
    if 8 in failed:  # the wall-clock race only, never the FLOP identity
        assert "not faster than full" in out, out


DROPIN_CHECK = os.path.join(ROOT, "paper_2509_09682_b200", "shim", "build", "dropin_check")


@pytest.mark.parametrize("dtype", ["f64", "f32", "bf16"])
def test_dropin_reference_api_parity_every_dtype(cuda, dtype):
    """The drop-in through the reference's own API in every device dtype:
    lseforge::cce_forward / cce_backward / ccem_forward / ccem_backward (the
    shim: lf_convert_rows, lf_classifier_to_items, the kernels,
    lf_widen_grad, lf_items_grad_to_classifier) vs the reference's
    materialising oracles (losses.cpp, linked unchanged) at the stated
    per-dtype tolerances (tests/gpu_util.py TOL), on bf16-representable
    inputs so every dtype sees the same values."""
    if not os.path.exists(DROPIN_CHECK):
        pytest.skip(f"{DROPIN_CHECK} not built (needs /root/reference at build time)")
    env = dict(os.environ, LSEFORGE_B200_DTYPE=dtype)
    p = subprocess.run([DROPIN_CHECK, "parity"], capture_output=True, text=True, timeout=600, env=env)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and out.strip().endswith("OK") and "FAIL" not in out, out[-4000:]
