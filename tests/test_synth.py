"""Input generators (synth/): determinism, shape, and the paper's skew phenomenon."""
import numpy as np

from synth import configs, hashgen, traces


def test_walk_spike_deterministic_distinct_and_skewed():
    a = traces.walk_spike(16, 4096, 2, 12, seed=5)
    b = traces.walk_spike(16, 4096, 2, 12, seed=5)
    for (ia, ga), (ib, gb) in zip(a, b):
        assert np.array_equal(ia, ib) and np.array_equal(ga.view(np.uint32), gb.view(np.uint32))
        s = np.sort(ia, axis=1)
        assert (s[:, 1:] != s[:, :-1]).all()
        assert np.allclose(ga.sum(1), 1.0, atol=1e-6) and (ga > 0).all()
    # >16x swing of one expert's load within 3 iterations
    assert traces.max_swing(a, 16) >= 16


def test_rotating_hot_exact_16x():
    E, T, k = 64, 8192, 2
    tr = traces.rotating_hot(E, T, k, 7, seed=1)
    c = np.stack([traces.expert_counts(i, E) for i, _ in tr])
    assert (c.sum(1) == T * k).all()
    for ids, _ in tr:
        s = np.sort(ids, axis=1)
        assert (s[:, 1:] != s[:, :-1]).all()
    # the hot set moves every 3 iterations: an expert jumps ~16x
    assert traces.max_swing(tr, E) >= 15.9


def test_configs_shapes():
    for name, wl in configs.CONFIGS.items():
        G = wl.G_default
        S = wl.S(G)
        assert wl.P % G == 0 and (wl.P // G) % 8 == 0, name
        assert wl.E <= S * G
        wl.tokens_per_rank(G)
    assert configs.CONFIGS["gpt-small"].P == 8_388_608
    assert configs.CONFIGS["mixtral"].P == 176_160_768
    assert configs.CONFIGS["qwen3-fine"].P == 4_718_592


def test_hash_values_are_exact_bit_constructions():
    g = hashgen.grad_bits(1, 2, 3, np.arange(100_000, dtype=np.uint64))
    expo = (g >> 7) & 0xFF
    assert expo.min() >= 112 and expo.max() <= 123
    assert len(np.unique(expo)) == 12
    m = hashgen.master_bits(1, 2, np.arange(100_000, dtype=np.uint64))
    e32 = (m >> 23) & 0xFF
    assert e32.min() >= 119 and e32.max() <= 123
    # counter-based: any index subset gives the same values as the full range
    idx = np.array([7, 99_999, 0], dtype=np.uint64)
    assert np.array_equal(hashgen.grad_bits(1, 2, 3, idx), g[idx.astype(np.int64)])
    # known value (regression pin for the CUDA twin in csrc/synth.cu)
    assert int(hashgen.splitmix64(np.array([0], np.uint64))[0]) == 0xE220A8397B1DCDAF
