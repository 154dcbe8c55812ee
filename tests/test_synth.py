"""The C column-chunk generator (synth/csynth.c) reproduces synth/generators.py
bit for bit -- it feeds the streamed oracle of the full-size parity tests."""
import numpy as np

import synth
from synth import fast


def test_linear_cols_bit_identical():
    K, N = 512, 384
    q, z, s = synth.gen_linear(3, 5, synth.KIND["WGATE"], K, N)
    for n0, n1 in [(0, N), (7, 100), (256, 384)]:
        qc, zc, sc = fast.gen_linear_cols(3, 5, synth.KIND["WGATE"], K, N, n0, n1)
        assert np.array_equal(qc, q[:, n0:n1]) and np.array_equal(zc, z[:, n0:n1]) and np.array_equal(sc, s[:, n0:n1])


def test_rows_and_prefix_bit_identical():
    h, V = 256, 1000
    rows = [0, 3, 999, 512]
    assert np.array_equal(fast.gen_embed_rows(1, h, rows), synth.gen_embed(1, V, h, rows=np.array(rows)))
    assert np.array_equal(fast.gen_lm_head_rows(1, h, rows), synth.gen_lm_head(1, V, h, rows=np.array(rows)))
    k, v = synth.gen_prefix_kv(2, 1, 70, 4, 64)
    kf, vf = fast.gen_prefix_kv(2, 1, 70, 4, 64)
    assert np.array_equal(k, kf) and np.array_equal(v, vf)
