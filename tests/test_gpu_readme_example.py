"""The README's usage example, at a smaller P, so the documented API stays runnable."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_readme_usage_example():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2504_19925_b200 import (DecoupledExpertLayer, MOE_TOK_GATE, TokenExchange,
                                       moe_slot_capacity, moe_token_combine, moe_token_dispatch)
    from synth import traces
    torch.cuda.set_device(0)
    E, G, S, k, P, T, d = 16, 1, 64, 2, 8 * 1024, 4096, 1024
    layer = DecoupledExpertLayer(E=E, G=G, S=S, k=k, P=P, max_tokens=T, rank=0, device=0, seed=0,
                                 capacity=moe_slot_capacity(2.0, T, k, G, S))
    ids_np, gates_np = traces.walk_spike(E, T, k, 1, seed=3)[0]
    ids, gates = torch.from_numpy(ids_np).cuda(), torch.from_numpy(gates_np).cuda()
    plan_next = layer.iterate(ids, gates, T)
    layer.sync_weights()
    assert int(plan_next.replicas.sum()) == G * S
    assert layer.out.counts_host.sum().item() == T * k
    tx = TokenExchange(layer.ctx, d=d, rows=layer.out.capacity)
    x = torch.randn(T * d, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    moe_token_dispatch(tx, [x], T, layer.out)
    moe_token_combine(tx, [y], T, layer.out, gates=gates, flags=MOE_TOK_GATE)
    layer.ctx.check()
    # identity "expert": y = sum over kept pairs of gate * x (gates of a token sum to <= 1)
    kept = (layer.out.dest_slot.view(T, k) >= 0).float()
    want = (x.float().view(T, 1, d) * (gates * kept).view(T, k, 1)).sum(1)
    assert torch.allclose(y.float().view(T, d), want, atol=0.02, rtol=0.02)
    tx.close()
    layer.close()
