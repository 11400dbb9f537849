"""The experiment switches DESIGN.md lists keep the results exact: each runs
tests/ab_check.py (C2 LUT re-test frames joined and pipelined, C3) in its own
process with the switch set, against the oracle."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("switch", [
    {"FIZI_FIX_OLD": "1"},                 # round 1's LUT re-test kernel
    {"FIZI_INLINE": "1"},                  # per-pixel words inside the fused kernel
    {"FIZI_MASK_MODE": "zero"},            # round 1's mask clear + kept-run writes
    {"FIZI_NO_GRAPH": "1"},                # direct launches instead of graph replays
    {"FIZI_SEG_PERSIST": "0"},             # one CTA per work item
    {"FIZI_GROUP": "8"},                   # frames per work item
    {"FIZI_MULTI_CFG": "1", "FIZI_SLOW_GRID": "3"},
])
def test_experiment_switch_is_exact(switch):
    env = dict(os.environ, **switch)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "ab_check.py")],
                       capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), (switch, r.stdout[-2000:],
                                                                   r.stderr[-3000:])
