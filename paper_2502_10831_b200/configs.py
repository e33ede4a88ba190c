"""Workload definitions: BASELINE.json ``configs`` as seeded synthetic inputs.

No public dataset is involved; the reference's own protocol (SPEC.md:367-380,
PAPER.md:240) is SplitMix64 from seed 2024873, which K4 reproduces in counter
form.  Each config gets its own stream seed (PAPER_SEED + id) so the arrays do
not overlap.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

PAPER_SEED = 2024873
UNIFORM, TAN_STRESS = 0, 1
SIN, COS, TAN = 1, 2, 4


@dataclass(frozen=True)
class Workload:
    name: str
    dtype: str  # "float32" | "float64"
    n: int
    dist: int
    lo: float
    hi: float
    seed: int
    mask: int
    kind: int = 0  # 0 proposed, 1 taylor
    n_terms: int = 5
    note: str = ""

    @property
    def itemsize(self) -> int:
        return 4 if self.dtype == "float32" else 8

    @property
    def bytes_per_elem(self) -> int:
        """Algorithmic HBM bytes per element: read x once + write each output once."""
        return self.itemsize * (1 + bin(self.mask).count("1"))


TWO_PI = 2.0 * math.pi

CONFIGS = {
    # configs[0]: fp32, 2^24, U[0, 2pi), three separate outputs
    "cfg1": Workload("cfg1", "float32", 1 << 24, UNIFORM, 0.0, TWO_PI, PAPER_SEED + 1, 7,
                     note="fp32 2^24 U[0,2pi) proposed sin/cos/tan, three output arrays"),
    # configs[1]: fp64, 2^28, U[-1000pi, 1000pi], fused S/C/T  (the bench workload)
    "cfg2": Workload("cfg2", "float64", 1 << 28, UNIFORM, -1000.0 * math.pi, 1000.0 * math.pi,
                     PAPER_SEED + 2, 7,
                     note="fp64 2^28 U[-1000pi,1000pi] fused proposed sin/cos/tan"),
    # configs[2]: tan stress, fp32, 2^26, x = (2k+1) pi/2 + delta
    "cfg3": Workload("cfg3", "float32", 1 << 26, TAN_STRESS, -1000.0, 1000.0, PAPER_SEED + 3, 4,
                     note="fp32 2^26 tan stress: (2k+1)pi/2 + N(0,1e-3) clipped to 0.05"),
    # configs[3]: Taylor-5 sin/cos, fp32 and fp64, 2^28, U[0, 2pi)
    "cfg4_f32": Workload("cfg4_f32", "float32", 1 << 28, UNIFORM, 0.0, TWO_PI, PAPER_SEED + 4, 3,
                         kind=1, n_terms=5, note="Taylor-5 sin/cos fp32 2^28 U[0,2pi)"),
    "cfg4_f64": Workload("cfg4_f64", "float64", 1 << 28, UNIFORM, 0.0, TWO_PI, PAPER_SEED + 4, 3,
                         kind=1, n_terms=5, note="Taylor-5 sin/cos fp64 2^28 U[0,2pi)"),
    # configs[4]: 8-GPU sharded sweep, fp32 2^33 U[-100pi, 100pi], fused S/C/T
    "cfg5": Workload("cfg5", "float32", 1 << 33, UNIFORM, -100.0 * math.pi, 100.0 * math.pi,
                     PAPER_SEED + 5, 7,
                     note="fp32 2^33 U[-100pi,100pi] fused, contiguous shards per GPU"),
}

# The paper's own accuracy protocol: 1000 angles in [-1e6, 1e6), seed 2024873
# (PAPER.md:240).
PAPER_PROTOCOL = Workload("paper", "float64", 1000, UNIFORM, -1e6, 1e6, PAPER_SEED, 7,
                          note="PAPER.md:240 1000 angles in +-1e6")


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous equal shard [lo, hi) of n elements for `rank` of `world`."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi
