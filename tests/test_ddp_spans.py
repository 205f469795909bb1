"""Host-side logic of the DDP hook on CPU: splitting a flat
gradient bucket into APS layers at its parameter boundaries, merging a parameter whose
view would not start 16-byte aligned into the preceding layer (several
consecutive layers may be treated "as a whole tensor").  The spans must tile the bucket
exactly, every span must start 16-byte aligned, and a parameter is merged only when its
own start is misaligned."""
import numpy as np
import pytest
import torch

from paper_1911_08907_b200.ddp import layer_spans


def _check(buf, numels):
    spans, groups = layer_spans(buf, numels)
    # the spans tile [0, sum(numels)) in order, and the groups partition the parameters in order
    off = 0
    for (o, n) in spans:
        assert o == off and n > 0
        assert (buf.data_ptr() + 4 * o) % 16 == 0, "every APS layer starts 16-byte aligned"
        off += n
    assert off == sum(numels)
    assert [i for g in groups for i in g] == list(range(len(numels)))
    starts = np.concatenate([[0], np.cumsum(numels)[:-1]])
    for g, (o, n) in zip(groups, spans):
        assert sum(numels[i] for i in g) == n and starts[g[0]] == o
        for i in g[1:]:  # merged only because its own start is misaligned
            assert (buf.data_ptr() + 4 * int(starts[i])) % 16 != 0
    return spans, groups


def test_aligned_parameters_stay_separate():
    numels = [4096, 64, 64, 36864, 256, 1000, 4]
    buf = torch.zeros(sum(numels), dtype=torch.float32)
    spans, groups = _check(buf, numels)
    assert len(spans) == len(numels)


def test_misaligned_parameters_merge():
    numels = [37 * 129, 129, 129 * 515, 515, 3 * 515, 3, 3, 3]
    buf = torch.zeros(sum(numels), dtype=torch.float32)
    spans, groups = _check(buf, numels)
    assert len(spans) < len(numels)


@pytest.mark.parametrize("seed", range(20))
def test_random_bucket_layouts(seed):
    rng = np.random.default_rng(seed)
    numels = [int(x) for x in rng.integers(1, 5000, rng.integers(1, 40))]
    base = torch.zeros(sum(numels) + 8, dtype=torch.float32)
    for shift in range(4):  # the bucket's own start at 0, 4, 8, 12 bytes past a 16-byte boundary
        buf = base[shift:shift + sum(numels)]
        if buf.data_ptr() % 16 == 0 or shift:
            spans, _ = layer_spans(buf, numels)
            if buf.data_ptr() % 16 == 0:
                _check(buf, numels)
            else:  # a misaligned bucket start: the first layer still starts at offset 0
                assert spans[0][0] == 0 and sum(n for _, n in spans) == sum(numels)
