"""The hand-written counting sort (csrc/sort.cu) against numpy's stable argsort.

mdkk_bucket_sort replaces the reference's `np.argsort(cid, kind="stable")` +
`np.bincount` + `cumsum` binning (mdkk/neighbor.py:88-96) and the owner
partition of migrate (mdkk/domain.py:324-334): the order must be exactly the
stable one (rows ascending within a bucket) and the starts the cumulative
counts, for many buckets (cells) and few (ranks), including empty buckets,
heavy buckets and n not a multiple of the block sizes.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sort(keys: np.ndarray, nb: int):
    import torch
    from paper_2508_13523_b200 import _lib
    dev = torch.device("cuda", 0)
    k = torch.from_numpy(keys.astype(np.int32)).to(dev)
    start = torch.full((nb + 1,), -7, dtype=torch.int32, device=dev)
    order = torch.full((max(len(keys), 1),), -7, dtype=torch.int32, device=dev)
    _lib.call("mdkk_bucket_sort", _lib.ctx(dev), k.data_ptr(), len(keys), nb, start.data_ptr(), order.data_ptr(),
              _lib.stream(dev))
    return start.cpu().numpy(), order[: len(keys)].cpu().numpy()


@pytest.mark.parametrize("n,nb,seed", [(1, 1, 0), (257, 3, 1), (100_003, 8, 2), (65_536, 64, 3),
                                       (2_000_001, 125_000, 4), (50_000, 70, 5), (30_000, 1 << 20, 6)])
def test_bucket_sort_is_the_stable_argsort(gpu, n, nb, seed):
    rng = np.random.default_rng(seed)
    keys = rng.integers(0, nb, n)
    start, order = _sort(keys, nb)
    assert np.array_equal(order, np.argsort(keys, kind="stable"))
    assert np.array_equal(start, np.concatenate([[0], np.cumsum(np.bincount(keys, minlength=nb))]))


def test_bucket_sort_heavy_and_empty_buckets(gpu):
    rng = np.random.default_rng(9)
    keys = np.concatenate([np.full(5000, 17), rng.integers(0, 1000, 20000), np.full(40, 999)])
    rng.shuffle(keys)
    start, order = _sort(keys, 1000)
    assert np.array_equal(order, np.argsort(keys, kind="stable"))
    start0, _ = _sort(np.zeros(0, np.int64), 5)
    assert np.array_equal(start0, np.zeros(6))
