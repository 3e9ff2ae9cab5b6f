"""The device generator (gen/csrc/gen.cu) reproduces gen/inputs.py byte for byte."""
import numpy as np
import pytest
import torch

from gen import device as gdev
from gen import inputs as gen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [
    dict(kind=gen.DELTA, m=32, delta=(1 << 32) // 32, dist=gen.DIST_UNIFORM),
    dict(kind=gen.DELTA, m=7, delta=-(-(1 << 32) // 7), dist=gen.DIST_SKEW, alpha=0.1),
    dict(kind=gen.IDENTITY, m=256, dist=gen.DIST_UNIFORM),
    dict(kind=gen.IDENTITY, m=200, dist=gen.DIST_BINOMIAL),
    dict(kind=gen.RADIX, m=64, shift=5, bits=6, dist=gen.DIST_SKEW, alpha=0.0),
    dict(kind=gen.RADIX, m=256, shift=24, bits=8, dist=gen.DIST_BINOMIAL),
])
def test_device_generator_matches_host(cfg):
    n = 300001
    h = gen.keys(n, seed=123, **cfg)
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    gdev.keys_(d, 123, **cfg)
    assert np.array_equal(d.cpu().numpy().view(np.uint32), h)
    for parity in (True, False):
        gdev.values_(d, 77, parity=parity)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), gen.values(n, 77, parity=parity))
