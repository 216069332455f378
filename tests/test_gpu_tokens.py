"""GPU parity of row f3 (token all-to-all, include/moe_tokens.h) against oracle/tokens.py:
every written expert-buffer row and every combined token, bit for bit, over several
iterations of a trace, with and without capacity drops and gate weighting."""
import numpy as np
import pytest
import torch

from synth import configs, traces

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()
    torch.cuda.set_device(0)


def _plan_from_oracle(p, G, S):
    """The oracle's placement (replicas, first_slot, slot_expert) as a moe_plan_t for the layer."""
    from paper_2504_19925_b200 import api
    E = len(p["replicas"])
    pl = api.Plan(E, G, S)
    pl.replicas[:] = p["replicas"]
    pl.first_slot[:] = p["first_slot"]
    pl.slot_expert[:] = p["slot_expert"]
    return pl


def _bits(rng, shape):
    """bf16 bit patterns of N(0, 1) values (inputs only; no method arithmetic)."""
    from oracle.numerics import f32_to_bf16_rne
    return f32_to_bf16_rne(rng.normal(size=shape).astype(np.float32))


def _to_dev(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(bits.view(np.int16).copy()).cuda().view(torch.bfloat16)


def _from_dev(t: torch.Tensor) -> np.ndarray:
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def run_tokens(name, G: int, iters: int, cf: float = 0.0, flags: int = 0, T: int | None = None,
               seed: int | None = None):
    from paper_2504_19925_b200 import DecoupledExpertLayer, TokenExchange, api
    from oracle import dispatch as OD
    from oracle import plan as OP
    from oracle import tokens as OT
    wl = configs.CONFIGS[name] if isinstance(name, str) else name
    if seed is None:
        seed = configs.seed_for(wl.name)
    S, E, k, d = wl.S(G), wl.E, wl.k, wl.d
    TT = wl.T if T is None else T
    Tg = TT // G
    cap = OD.slot_capacity(cf, TT, k, G * S) if cf > 0 else 0
    tr = traces.make_trace(wl, iters=iters, T=TT, seed=seed)
    # oracle routing for every iteration first (it sizes the buffers)
    plan = OP.plan(np.ones(E, np.int64), E, G, S)
    routes = []
    for ids, gates in tr:
        disp = OD.dispatch(traces.split_ranks(ids, G), traces.split_ranks(gates, G), plan["first_slot"], E, cap)
        routes.append((plan, disp))
        plan = OP.plan(disp["C"], E, G, S)
    rows = max(1, max(int(dp["slot_load"].max()) for _, dp in routes))
    layer = DecoupledExpertLayer(E, G, S, k, 8 * G, Tg, rank=-1, device=0, seed=1, capacity=cap)
    tx = TokenExchange(layer.ctx, d, rows)
    rng = np.random.default_rng(seed + 17)
    use_gate = bool(flags & api.MOE_TOK_GATE)
    for it, ((ids, gates), (plan_t, disp)) in enumerate(zip(tr, routes)):
        layer.plan = _plan_from_oracle(plan_t, G, S)
        ids_d = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
        gates_d = torch.from_numpy(np.ascontiguousarray(gates)).cuda()
        layer.dispatch(ids_d, gates_d, Tg)
        xs = [_bits(rng, (Tg, d)) for _ in range(G)]
        src = [_to_dev(x) for x in xs]
        api.moe_token_dispatch(tx, src, Tg, layer.out, gates=gates_d, flags=flags)
        layer.ctx.check()
        want = np.zeros((G * S, rows, d), np.uint16)
        for g in range(G):
            rk = disp["ranks"][g]
            OT.token_dispatch(xs[g], rk["dest_slot"], rk["dest_off"], want,
                              gates=traces.split_ranks(gates, G)[g].reshape(-1) if use_gate else None)
        for h in range(G):
            got = _from_dev(tx.slot_view(h))
            for ls in range(S):
                n = int(disp["slot_load"][h * S + ls])
                assert np.array_equal(got[ls, :n], want[h * S + ls, :n]), f"iter {it}: slot {h * S + ls} rows"
        # the "expert": overwrite every buffer with synthetic outputs, then combine
        y = _bits(rng, (G * S, rows, d))
        for h in range(G):
            tx.slot_view(h).copy_(_to_dev(y[h * S:(h + 1) * S]).view(S, rows, d))
        dst = [torch.empty(Tg * d, dtype=torch.bfloat16, device="cuda") for _ in range(G)]
        api.moe_token_combine(tx, dst, Tg, layer.out, gates=gates_d, flags=flags)
        layer.ctx.check()
        for g in range(G):
            rk = disp["ranks"][g]
            exp = OT.token_combine(y, rk["dest_slot"], rk["dest_off"], Tg,
                                   gates=traces.split_ranks(gates, G)[g].reshape(-1) if use_gate else None)
            assert np.array_equal(_from_dev(dst[g]).reshape(Tg, d), exp), f"iter {it} rank {g}: combine"
    tx.close()
    layer.close()


@pytest.mark.parametrize("name,G,cf,flags", [("tiny-skew", 4, 0.0, 0), ("tiny-skew", 4, 0.0, 1),
                                             ("tiny-odd", 3, 0.5, 1), ("tiny", 2, 1.0, 0),
                                             ("medium", 4, 1.25, 1), ("medium", 1, 0.0, 0)])
def test_token_dispatch_and_combine_virtual(name, G, cf, flags):
    run_tokens(name, G, 3, cf=cf, flags=flags)


def test_token_exchange_gpt_small_full_size():
    """BASELINE's GPT-MoE small shape (d = 1024, T = 65 536, k = 2) at G = 1 and 8."""
    run_tokens("gpt-small", 1, 1, flags=1)
    run_tokens("gpt-small", 8, 1, cf=1.0, flags=0)


def test_token_rows_overflow_raises():
    from paper_2504_19925_b200 import DecoupledExpertLayer, MoeError, TokenExchange, api
    layer = DecoupledExpertLayer(8, 1, 8, 2, 64, 128, rank=0, device=0)
    ids = torch.stack([torch.zeros(128, dtype=torch.int32), torch.ones(128, dtype=torch.int32)], 1).cuda()
    gates = torch.ones((128, 2), dtype=torch.float32, device="cuda")
    layer.dispatch(ids, gates, 128)
    tx = TokenExchange(layer.ctx, 16, 4)       # expert 0 alone gets 128 rows > 4
    x = torch.zeros(128 * 16, dtype=torch.bfloat16, device="cuda")
    api.moe_token_dispatch(tx, [x], 128, layer.out)
    with pytest.raises(MoeError) as ei:
        layer.ctx.check()
    assert ei.value.status == 3
    with pytest.raises(MoeError):
        TokenExchange(layer.ctx, 12, 4)          # d % 8 != 0
    tx.close()
    layer.close()


def test_special_values_bitwise():
    """NaN payloads, +-Inf, denormals, signed zeros and fp32 rounding ties through the copy
    dispatch (bits preserved) and the combine (fp32 sum -> bf16 RNE, NaN -> 0x7FFF, A17)."""
    from paper_2504_19925_b200 import DecoupledExpertLayer, TokenExchange, api
    from oracle import dispatch as OD
    from oracle import plan as OP
    from oracle import tokens as OT
    E, G, S, k, T, d = 4, 1, 4, 2, 64, 64
    rng = np.random.default_rng(3)
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    gates = rng.choice(np.array([1.0, 0.5, 3.0, 1e-30, -2.0, 1.0000001], np.float32), size=(T, k))
    special = np.array([0x7FC0, 0xFFC1, 0x7F80, 0xFF80, 0x0001, 0x8001, 0x0000, 0x8000, 0x3F81, 0x7F7F,
                        0x4B80, 0xCB80, 0x3F80, 0x0080], np.uint16)
    x = rng.choice(special, size=(T, d)).astype(np.uint16)
    plan = OP.plan(np.ones(E, np.int64), E, G, S)
    disp = OD.dispatch([ids], [gates], plan["first_slot"], E)
    rows = int(disp["slot_load"].max())
    layer = DecoupledExpertLayer(E, G, S, k, 8, T, rank=0, device=0)
    layer.plan = _plan_from_oracle(plan, G, S)
    gates_d = torch.from_numpy(gates).cuda()
    layer.dispatch(torch.from_numpy(ids).cuda(), gates_d, T)
    tx = TokenExchange(layer.ctx, d, rows)
    for flags in (0, 1):
        api.moe_token_dispatch(tx, [_to_dev(x)], T, layer.out, gates=gates_d, flags=flags)
        want = np.zeros((S, rows, d), np.uint16)
        OT.token_dispatch(x, disp["ranks"][0]["dest_slot"], disp["ranks"][0]["dest_off"], want,
                          gates=gates.reshape(-1) if flags else None)
        got = _from_dev(tx.slot_view(0))
        for s in range(S):
            n = int(disp["slot_load"][s])
            assert np.array_equal(got[s, :n], want[s, :n]), (flags, s)
        dst = torch.empty(T * d, dtype=torch.bfloat16, device="cuda")
        api.moe_token_combine(tx, [dst], T, layer.out, gates=gates_d, flags=flags)
        exp = OT.token_combine(want, disp["ranks"][0]["dest_slot"], disp["ranks"][0]["dest_off"], T,
                               gates=gates.reshape(-1) if flags else None)
        assert np.array_equal(_from_dev(dst).reshape(T, d), exp), flags
    layer.ctx.check()
    tx.close()
    layer.close()


def test_context_close_closes_token_exchange_first():
    """Closing the context first must not leave a dangling token exchange (use-after-free)."""
    from paper_2504_19925_b200 import DecoupledExpertLayer, TokenExchange
    layer = DecoupledExpertLayer(8, 1, 8, 2, 64, 16, rank=0, device=0)
    tx = TokenExchange(layer.ctx, 16, 4)
    layer.close()                      # closes tx, then the context
    assert tx._h is None
    tx.close()                         # idempotent


@pytest.mark.parametrize("case", range(40))
def test_token_exchange_fuzz(case):
    """Random E (from 1), G (to 8), S, k (to E), T (ragged, from 0), d (multiple of 8, also
    not a multiple of the kernels' 128/256-vector chunks), capacity and gate flags."""
    from oracle.dispatch import slot_capacity
    rng = np.random.default_rng(5000 + case)
    G = int(rng.choice([1, 2, 3, 4, 8]))
    E = int(rng.integers(1, 20))
    S = -(-E // G) + int(rng.integers(0, 4))
    k = int(rng.integers(1, min(E, 5) + 1))
    T = G * int(rng.integers(0, 200)) if case % 8 else 0
    d = 8 * int(rng.integers(1, 160))
    wl = configs.Workload(f"tfuzz{case}", E=E, d=d, ffn=1, mats=1, k=k, T=T, slots_total=G * S,
                          trace="walk-spike", G_default=G)
    cf = float(rng.uniform(0.3, 2.0)) if rng.random() < 0.4 else 0.0
    run_tokens(wl, G, 2, cf=cf, flags=int(rng.integers(0, 2)), seed=900 + case)
