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


def test_edge_generators_cover_their_categories():
    """synth/edge.py: deterministic bit patterns; every category is present."""
    from synth import edge
    idx = np.arange(1 << 16, dtype=np.uint64)
    g = edge.edge_grad_bits(4, 2, 9, idx)
    assert np.array_equal(g, edge.edge_grad_bits(4, 2, 9, idx))
    ex, mant = (g >> 7) & 0xFF, g & 0x7F
    assert (g == 0).any() and (g == 0x8000).any()
    assert ((ex == 0) & (mant != 0)).any()                       # denormals
    assert ((ex >= 200) & (ex < 248)).any() and (ex == 254).any()
    assert ((g & 0x7FFF) == 0x7F80).any()                        # +-inf
    assert ((ex == 255) & (mant != 0)).any()                     # NaN
    m = edge.edge_master_bits(4, 3, idx)
    mex = (m >> 23) & 0xFF
    assert (m == 0).any() and (m == 0x80000000).any() and ((mex == 0) & (m & 0x7FFFFF != 0)).any()
    assert ((m & 0xFFFF) == 0x8000).any()                        # bf16 ties
    assert ((mex == 254) & ((m & 0x7F8000) == 0x7F8000)).any()   # RNE to bf16 overflows


def test_idle_expert_trace_and_zero_slots():
    from synth import edge
    E, T, k = 8, 512, 2
    tr = edge.idle_expert_trace(E, T, k, 6, seed=3)
    idle_counts = []
    for ids, gates in tr:
        s = np.sort(ids, axis=1)
        assert (s[:, 1:] != s[:, :-1]).all() and (gates > 0).all() and (gates <= 1).all()
        c = np.bincount(ids.reshape(-1), minlength=E)
        idle_counts.append(int((c == 0).sum()))
        slot_expert = np.repeat(np.arange(E), 2)                 # 2 slots per expert
        zs = edge.zero_slots(ids, E, slot_expert)
        want = [j for j in range(2 * E) if c[slot_expert[j]] == 0]   # brute force
        assert zs.tolist() == want
    assert idle_counts[0] == E - k and max(idle_counts) >= E - k and min(idle_counts) >= 1


def test_trace_iterations_are_independent_and_pool_identical():
    """make_trace(workers>1) and the per-iteration generators give exactly the sequential
    arrays (the recipe of DESIGN.md §4 is unchanged by parallel generation)."""
    wl = configs.CONFIGS["tiny-skew"]
    seq = traces.make_trace(wl, iters=7)
    par = traces.make_trace(wl, iters=7, workers=3)
    for (a, ga), (b, gb) in zip(seq, par):
        assert np.array_equal(a, b) and np.array_equal(ga.view(np.uint32), gb.view(np.uint32))
    ids5, g5 = traces.walk_spike_iter(wl.E, wl.T, wl.k, 5, configs.seed_for(wl.name))
    assert np.array_equal(ids5, seq[5][0]) and np.array_equal(g5, seq[5][1])
    st = configs.CONFIGS["stress"]
    a = traces.make_trace(st, iters=4, T=4096)
    b = traces.make_trace(st, iters=4, T=4096, workers=2)
    assert all(np.array_equal(x[0], y[0]) for x, y in zip(a, b))
