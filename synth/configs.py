"""Concrete workloads for the BASELINE.json configs.

BASELINE.json ``configs`` list five workloads; SURVEY.md §8(d).1 turns them into
shapes.  Readings:

* A13 -- slots per GPU are not given by the paper (except ``tiny``); the total
  number of slots S*G is fixed per config so that the same workload runs at
  G = 1, 2, 4, 8 (strong scaling).  GPT-small uses the paper's 4x average
  replication (16 experts, 64 instances).
* A14 -- P = n_mats * d * ffn parameters per expert (no biases); n_mats = 2 for
  GPT-style experts and 3 for SwiGLU experts (Mixtral, Qwen).
* A21 -- rank g owns the contiguous token block [g*T/G, (g+1)*T/G).

``tiny-skew`` and ``tiny-odd`` are parity-only variants: ``tiny`` itself is
degenerate (E == S*G, so every expert always has exactly one replica).
``tiny-odd`` has a ragged element range per owner (P/G not a multiple of the
kernel chunk) and a ragged pair count per rank (not a multiple of the tile).
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    E: int            # expert classes
    d: int            # model dim
    ffn: int          # expert hidden dim
    mats: int         # weight matrices per expert (2 GPT-style, 3 SwiGLU)
    k: int            # top-k
    T: int            # global tokens per iteration
    slots_total: int  # S * G, fixed across G (reading A13)
    trace: str        # "walk-spike" | "rotating-hot"
    G_default: int    # G the config is quoted at
    iters: int = 20

    @property
    def P(self) -> int:
        """Parameters per expert (reading A14)."""
        return self.mats * self.d * self.ffn

    def S(self, G: int) -> int:
        if self.slots_total % G:
            raise ValueError(f"{self.name}: S*G={self.slots_total} not divisible by G={G}")
        return self.slots_total // G

    def tokens_per_rank(self, G: int) -> int:
        if self.T % G:
            raise ValueError(f"{self.name}: T={self.T} not divisible by G={G}")
        return self.T // G


CONFIGS = {
    "tiny": Workload("tiny", E=8, d=64, ffn=256, mats=2, k=2, T=4096, slots_total=8,
                     trace="walk-spike", G_default=4),
    "tiny-skew": Workload("tiny-skew", E=8, d=64, ffn=256, mats=2, k=2, T=4096, slots_total=16,
                          trace="walk-spike", G_default=4),
    "tiny-odd": Workload("tiny-odd", E=5, d=40, ffn=264, mats=2, k=2, T=4095, slots_total=6,
                         trace="walk-spike", G_default=3),
    "gpt-small": Workload("gpt-small", E=16, d=1024, ffn=4096, mats=2, k=2, T=65536,
                          slots_total=64, trace="walk-spike", G_default=8),
    "mixtral": Workload("mixtral", E=64, d=4096, ffn=14336, mats=3, k=2, T=262144,
                        slots_total=128, trace="walk-spike", G_default=8),
    "qwen3-fine": Workload("qwen3-fine", E=128, d=2048, ffn=768, mats=3, k=8, T=524288,
                           slots_total=256, trace="walk-spike", G_default=8),
    "stress": Workload("stress", E=64, d=1024, ffn=4096, mats=2, k=2, T=65536, slots_total=128,
                       trace="rotating-hot", G_default=8),
    # parity-only: GPT-small's shape scaled down so the oracle can check every element
    "medium": Workload("medium", E=16, d=256, ffn=2048, mats=2, k=2, T=16384, slots_total=64,
                       trace="walk-spike", G_default=4),
}

# BASE seed; config i uses BASE_SEED + i
BASE_SEED = 250419925


def seed_for(name: str) -> int:
    return BASE_SEED + list(CONFIGS).index(name)
