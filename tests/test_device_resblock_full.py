"""Tier-B parity at every BASELINE IEP config at full size.

The device runs the whole BASELINE batch (cfg1: 64 programs, cfg2: 512
balanced trees at depths 4–8, cfg3: 4096 programs) and is compared with the
fp64 oracle (itself pinned to torch conv2d: test_oracle_resblock_torch.py):

* cfg1: all 64 rows;
* cfg2: 32 rows per depth, spread over the batch;
* cfg3: 128 rows spread over program size (smallest and largest included).

Stated tolerance: max|dev − ref| / max|ref| ≤ 1e-3 and per
element |dev − ref| ≤ 5e-3·(|ref| + rms(ref)).
"""
import numpy as np
import pytest

import parity_full as P

pytestmark = pytest.mark.gpu


def _check(dev, ref):
    e = P.errors(dev, ref)
    assert np.isfinite(dev).all()
    assert e["max_norm"] <= P.TOL_NORM, e
    assert e["elem"] <= P.TOL_ELEM, e
    return e


def test_cfg1_all_rows_match_oracle():
    rows, dev, ref, sizes, st = P.run_config("cfg1", 64)
    assert rows == list(range(64))
    _check(dev, ref)
    assert st.expensive_calls == 232  # SURVEY §8(c) golden count


@pytest.mark.parametrize("depth", [4, 5, 6, 7, 8])
def test_cfg2_sampled_rows_match_oracle(depth):
    rows, dev, ref, sizes, st = P.run_config("cfg2", 32, depth=depth)
    assert len(rows) == 32 and (sizes == 2 ** depth - 1).all()
    _check(dev, ref)
    assert st.steps == depth and st.expensive_calls == 20 * (depth - 1)


def test_cfg3_sampled_rows_match_oracle():
    rows, dev, ref, sizes, st = P.run_config("cfg3", 128)
    assert len(rows) == 128 and sizes.max() == 16 and sizes.min() == 8
    _check(dev, ref)
    assert st.expensive_calls == 469
