"""Every rank mode of the m <= 32 postscan (kf_meta RANK, ms_meta.cuh) and both
store structures (producer warp or not) are bit-exact against the oracle; and
the hardware property the default mode relies on (lane-ordered shared-memory
increments, probed by ms_lane_ordered_increment) holds on this GPU."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def test_lane_ordered_increment_probe():
    ms = pytest.importorskip("paper_1701_01189_b200")
    assert ms._lib.load().ms_lane_ordered_increment() == 1


@pytest.mark.parametrize("rank", ["atomic", "ballot", "mix3", "mix2", "xatomic", "xmix3", "xmix2", "xpair", "inc"])
@pytest.mark.parametrize("prod", ["0", "1"])
def test_rank_mode_parity(rank, prod):
    env = dict(os.environ, MS_META_RANK=rank, MS_META_PROD=prod)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_rank_mode_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"MS_KF_REVERSE": "1", "MS_KM_KEEP": "4"}, {"MS_KF_PREFETCH": "0"},
                                 {"MS_KM_PREFETCH": "2"}, {"MS_NO_META": "1"}, {"MS_NO_RANK_INC": "1"},
                                 {"MS_NO_RUN_STORES": "1"}])
def test_pipeline_options_parity(env):
    """Measured-and-rejected or fallback pipeline options stay bit-exact."""
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "_rank_mode_check.py")], env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
