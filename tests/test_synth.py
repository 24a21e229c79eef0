"""The shared input generator: numpy and torch implementations are bit-identical; statistics are
the Irwin-Hall(12) recipe of DESIGN.md (mean ~0, variance ~1, |x| <= 6)."""
import numpy as np
import torch

import cqs_synth as S


def test_numpy_torch_bit_identical():
    a = S.numpy_values(20260418, 1, 12345, 5000)
    b = S.torch_values(20260418, 1, 12345, 5000).numpy()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_bf16_rounding_matches_torch():
    a = S.numpy_values(7, 2, 0, 4096)
    b = torch.from_numpy(a).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(S.round_bf16(a), b)


def test_statistics():
    x = S.numpy_values(3, 0, 0, 200000).astype(np.float64)
    assert abs(x.mean()) < 0.01 and abs(x.var() - 1.0) < 0.02 and np.abs(x).max() <= 6.0


def test_offsets_compose():
    full = S.numpy_values(5, 0, 0, 300)
    assert np.array_equal(full[100:200], S.numpy_values(5, 0, 100, 100))
    t = S.torch_tensor((1, 2, 5, 30), 5, "q").reshape(-1).numpy()
    assert np.array_equal(t, full)
