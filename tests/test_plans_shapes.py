"""The step inputs at the other BASELINE shapes, host side (no GPU needed): the
library's host sampler vs the reference (oracle/_ref) on the same seeds --
random_init state, k-means view clusters, the 8-view batch, every sampled pixel /
tile / weight of the plan (sample_plan.cpp:62-171,
view_sampler.cpp:101-184).  configs[2] is covered on the GPU box
(test_fullsize.py::test_cfg2_step_inputs_bit_exact); here configs[1], configs[4]
and configs[3]'s N = 13 / lane-width-1 sweep point."""
import numpy as np
import pytest

from test_fullsize import inputs


@pytest.mark.parametrize("shape", ["cfg1", "cfg3", "cfg4"])
def test_step_inputs_bit_exact(reflib, shape):
    from paper_2504_12905_b200 import splatlm
    from paper_2504_12905_b200.build import build
    build()
    H = splatlm.HostSampler()
    a = inputs(H, shape)
    b = inputs(reflib, shape)
    assert a[0] == b[0]
    assert [list(map(int, c)) for c in a[2]] == [list(map(int, c)) for c in b[2]]
    assert a[3] == b[3]
    pa, pb = a[4], b[4]
    assert pa.total_samples() == pb.total_samples() > 0
    for f in ("view_offset", "px", "py", "tile", "weight"):
        assert np.array_equal(getattr(pa, f), getattr(pb, f)), f
