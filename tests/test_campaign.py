"""The fault-injection campaign (campaign.py) runs the
same GPU path as the parity tests; its per-trial outcomes must equal the
oracle's for the same seeded flips, and Eq. 9 must be the plain l2 norm."""
import random

import numpy as np
import pytest
import torch

import campaign as CP
from tests.parity_util import assert_records_equal, oracle_run


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["none", "online", "offline", "offline_partial"])
def test_campaign_trials_equal_oracle(mode):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    R = CP.Runner()
    p = CP.problem("64x64x8", mode).replace(sweeps=32)
    rng = random.Random(5)
    for t in range(6):
        f = CP.random_flip(p, rng, bit=rng.choice([14, 22, 27, 30, 31]), max_sweep=32)
        g = R.run(p, [f])
        o = oracle_run(p, faults=[f])
        assert np.array_equal(g["u"].cpu().numpy().view(np.uint32), o["u"].view(np.uint32))
        assert_records_equal(dict(records=g["records"]), o)
        assert g["stats"]["detections"] == o["stats"]["detections"]


def test_l2_is_eq9():
    a = torch.tensor([[1.0, 2.0], [3.0, 4.0]])
    b = torch.tensor([[1.0, 0.0], [3.0, 1.0]])
    assert CP.l2(a, b) == pytest.approx(np.sqrt(4.0 + 9.0))
    assert CP.l2(a, torch.tensor([[float("inf"), 0.0], [0.0, 0.0]])) == float("inf")
    q = CP._q([1.0, 2.0, 3.0, 4.0, 5.0])
    assert q["median"] == 3.0 and q["q1"] == 2.0 and q["q3"] == 4.0 and q["max"] == 5.0
