"""The seeded input generators (workload/): the device-side twin of normal_bf16 draws the
same bits as the numpy one (so a GPU test can generate a W too large for numpy and the
oracle still sees exactly the generator's values)."""
import math

import numpy as np
import pytest
import torch

import workload


@pytest.mark.parametrize("rows,cols,row_start,std", [(3, 7, 0, 1.0), (40, 896, 5, 1.0 / math.sqrt(896)),
                                                     (2, 16384, 131071, 1.0 / 128.0)])
def test_normal_bf16_torch_matches_numpy(rows, cols, row_start, std):
    ref = workload.normal_bf16(9, workload.S_W, rows, cols, std, row_start=row_start)
    got = workload.normal_bf16_torch(9, workload.S_W, rows, cols, std, "cpu", row_start=row_start,
                                     chunk_elems=1000)
    assert np.array_equal(got.view(torch.int16).numpy().view(np.uint16), ref)


def test_normal_bf16_torch_counters_past_2_pow_32():
    """Counters (row * cols + col) beyond 2^32 -- the 2.5e9-element W of the int64-offset
    GPU test reaches 2.49e9; check a window far past it too."""
    start = (1 << 33) // 4096 + 3
    ref = workload.normal_bf16(4, workload.S_W, 2, 4096, 0.5, row_start=start)
    got = workload.normal_bf16_torch(4, workload.S_W, 2, 4096, 0.5, "cpu", row_start=start)
    assert np.array_equal(got.view(torch.int16).numpy().view(np.uint16), ref)
