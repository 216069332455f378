"""The bench's byte accounting (bench.update_stage_bytes) against closed forms and the oracle's
transfer-by-transfer count (CPU only)."""
import numpy as np

import bench
from oracle import plan as P
from oracle import step as ST


def test_plain_accounting_matches_closed_forms_and_oracle():
    rng = np.random.default_rng(3)
    for _ in range(100):
        G = int(rng.integers(1, 9))
        S = int(rng.integers(1, 9))
        E = int(rng.integers(1, G * S + 1))
        Pp = 8 * G * int(rng.integers(1, 4))
        fc = P.placement(P.alg1(rng.integers(0, 1000, size=E), E, G, S))[0]
        fn = P.placement(P.alg1(rng.integers(0, 1000, size=E), E, G, S))[0]
        hbm, nvl = bench.update_stage_bytes(fc, fn, G, S, Pp, E, dedup=False)
        # App. E: 2 phases x (sN - s)/N x 2P bytes per direction, for any placement
        assert nvl == 2 * (S * G - S) * (Pp // G) * 2
        vol = ST.nvlink_bytes(fc, fn, G, S, Pp)
        assert nvl == max(int((vol["reduce_recv"] + vol["place_recv"]).max()),
                          int((vol["reduce_sent"] + vol["place_sent"]).max()))
        if G == 1:
            assert hbm == 2 * S * Pp + 24 * E * Pp + 2 * S * Pp


def test_dedup_accounting_never_moves_more_nvlink_bytes():
    rng = np.random.default_rng(4)
    for _ in range(100):
        G = int(rng.integers(2, 9))
        S = int(rng.integers(1, 17))
        E = int(rng.integers(1, G * S + 1))
        Pp = 8 * G * 4
        c = (rng.pareto(1.0, size=E) * 100).astype(np.int64)
        fc = P.placement(P.alg1(c, E, G, S))[0]
        fn = P.placement(P.alg1(c[::-1].copy(), E, G, S))[0]
        _, plain = bench.update_stage_bytes(fc, fn, G, S, Pp, E, dedup=False)
        _, dd = bench.update_stage_bytes(fc, fn, G, S, Pp, E, dedup=True)
        assert dd <= plain


def test_per_gpu_lists_agree_with_the_maxima():
    """parts=True's per-GPU lists (used by tools/dedup_traffic.py for the virtual-mode ncu
    cross-check) are the terms the reported maxima are taken over; without de-dup there is no
    pre-sum or replication, and the plain per-GPU update bytes add up to the whole-job count."""
    rng = np.random.default_rng(5)
    for _ in range(100):
        G = int(rng.integers(1, 9))
        S = int(rng.integers(1, 17))
        E = int(rng.integers(1, G * S + 1))
        Pp = 8 * G * int(rng.integers(1, 4))
        c = (rng.pareto(1.0, size=E) * 100).astype(np.int64)
        fc = P.placement(P.alg1(c, E, G, S))[0]
        fn = P.placement(P.alg1(c[::-1].copy(), E, G, S))[0]
        for dedup in (False, True):
            b = bench.update_stage_bytes(fc, fn, G, S, Pp, E, dedup=dedup and G > 1, parts=True)
            assert b["update_hbm"] == max(b["update_per_gpu"])
            assert b["presum_hbm"] == max(b["presum_per_gpu"])
            assert b["replicate_hbm"] == max(b["replicate_per_gpu"])
            assert b["stage_hbm"] == max(u + p + r for u, p, r in
                                         zip(b["update_per_gpu"], b["presum_per_gpu"], b["replicate_per_gpu"]))
            if not (dedup and G > 1):
                assert sum(b["presum_per_gpu"]) == 0 and sum(b["replicate_per_gpu"]) == 0
                # every grad slice read once, every weight slice written once, state r+w once
                assert sum(b["update_per_gpu"]) == 2 * G * S * Pp + 24 * E * Pp + 2 * G * S * Pp
