"""The A/B variants kept behind environment switches (read once per process,
so each runs in a subprocess) stay parity-green: DSDE_STREAM=tma (TMA-fed
stream kernel), DSDE_TAIL=split (finalize / draw / select kernels) and
DSDE_TAIL=fused (one persistent kernel for the whole step). Each runs the
oracle-parity cases of test_gpu_verify.py that cover ragged tails, tiny V,
ld padding, k = 1 / 16 and device errors, plus dsde_step against the three
separate calls."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ("test_verify_parity or test_verify_ld_padding or test_verify_k1_and_k16 or "
         "test_device_errors or test_identical_rows or test_disjoint_one_hot or test_step_matches_three_calls")


@pytest.mark.parametrize("env", [{"DSDE_STREAM": "tma"}, {"DSDE_TAIL": "split"}, {"DSDE_TAIL": "fused"}],
                         ids=["stream_tma", "tail_split", "tail_fused"])
def test_variant_parity(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-k", CASES,
                        "tests/test_gpu_verify.py", "tests/test_gpu_signal.py"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
