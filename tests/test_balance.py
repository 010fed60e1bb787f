"""SURVEY §8e shard balancing (host logic, CPU): the LPT partition of a global batch's sequences
over G data-parallel ranks."""
import numpy as np
import pytest

import synth
from paper_2312_17482_b200.balance import imbalance, lpt_partition


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_lpt_partition_is_a_partition_with_equal_counts(G):
    lens = synth.make_lengths("lognormal", 4096, 128, synth.rng_for(11))
    parts = lpt_partition(lens, G)
    allidx = np.concatenate(parts)
    assert np.array_equal(np.sort(allidx), np.arange(4096))  # every sequence exactly once
    assert all(len(p) == 4096 // G for p in parts)
    assert all(np.all(np.diff(p) > 0) for p in parts)


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_lpt_balances_c5_nnz_below_half_a_percent(G, seed):
    """C5 (lognormal lengths, ~50 % pad): contiguous slices are off by ~1-3 %; LPT < 0.5 %."""
    lens = synth.make_lengths("lognormal", 4096, 128, synth.rng_for(100 + seed))
    lpt = imbalance(lens, lpt_partition(lens, G))
    contiguous = imbalance(lens, [np.arange(r * 4096 // G, (r + 1) * 4096 // G) for r in range(G)])
    assert lpt < 5e-3 and lpt <= contiguous


def test_lpt_uneven_counts_and_errors():
    lens = np.array([9, 8, 7, 1, 1, 1, 1])
    parts = lpt_partition(lens, 3, equal_counts=False)
    assert sorted(int(lens[p].sum()) for p in parts) == [9, 9, 10]
    with pytest.raises(ValueError):
        lpt_partition(lens, 3)  # 7 sequences do not split into 3 equal counts
    with pytest.raises(ValueError):
        lpt_partition(lens, 0)
