"""Oracle steps O1-O3: tile grid, execution order, waves, wave groups.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Pins (tests/test_oracle_plan.py): PAPER.md:235 (512 tiles / 128 SMs = 4 waves),
PAPER.md:378 (swizzle 2: tiles 0 and 2 finish in W1), PAPER.md:388 (reordered
indices of tiles 0 and 3 are 0 and 1), PAPER.md:370 (fig:signal counting
thresholds 2, 4, 2), PAPER.md:415 (partitions (1,2,2), (2,3) for T=5), plus
permutation / partition invariants.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import ceil

import numpy as np


class OracleError(ValueError):
    """Raised for inputs the method does not define (SURVEY.md §8(b) error list)."""


# ---------------------------------------------------------------- O1: tile grid
def tile_grid(M: int, N: int, BM: int, BN: int) -> tuple[int, int]:
    """O1 ("The output matrix C is partitioned into tiles").

    Returns (Mt, Nt).  Tile id t = i*Nt + j is tile-row i, tile-column j
    (row-major tile numbering).  Divisibility is required (R6)."""
    if M % BM or N % BN:
        raise OracleError(f"shape {M}x{N} not divisible by tile {BM}x{BN}")
    return M // BM, N // BN


def tile_coords(t: int, Nt: int) -> tuple[int, int]:
    return t // Nt, t % Nt


# ---------------------------------------------------------------- O2: order
def default_order(Mt: int, Nt: int, s: int) -> np.ndarray:
    """O2, default block swizzle of width s (
    DESIGN.md reading R1): row-panels of s tile-rows, panels top to bottom,
    and inside a panel the tiles are visited column by column (tile-row index
    fastest).  s = 1 is a row-major raster, s >= Mt is column-major."""
    if s < 1:
        raise OracleError("swizzle width must be >= 1")
    order = []
    for p0 in range(0, Mt, s):
        rows = range(p0, min(p0 + s, Mt))
        for j in range(Nt):
            for i in rows:
                order.append(i * Nt + j)
    return np.array(order, dtype=np.int64)


def validate_order(order, ntiles: int) -> np.ndarray:
    """An explicit order must be a permutation of 0..ntiles-1."""
    o = np.asarray(order, dtype=np.int64).reshape(-1)
    if o.size != ntiles or not np.array_equal(np.sort(o), np.arange(ntiles)):
        raise OracleError("tile order is not a permutation of the tile ids")
    return o


# ---------------------------------------------------------------- O3: waves & groups
def num_waves(ntiles: int, S: int) -> int:
    """T = ceil(#tiles / S) ("dividing tile number (512) by SM
    number (128)"; Alg. 1 line 3 with S = sm_num - comm sm_num)."""
    if S < 1:
        raise OracleError("wave width S must be >= 1")
    return ceil(ntiles / S)


def wave_of_position(p: int, S: int) -> int:
    """The tile at execution position p runs in wave floor(p / S)."""
    return p // S


def group_ranges(partition, S: int, ntiles: int) -> list[tuple[int, int]]:
    """Position ranges of the wave groups.

    Group j (0-based) holds the tiles at execution positions
    [S*W_{j-1}, min(S*W_j, ntiles)) where W_j = g_1 + ... + g_j (in waves)."""
    T = num_waves(ntiles, S)
    part = [int(g) for g in partition]
    if ntiles == 0 and part and all(g == 0 for g in part):
        # an All-to-All source with no rows (an expert no token was routed
        # to) still takes part in each of the P group exchanges, with empty
        # groups (the same P on every rank; R45)
        return [(0, 0)] * len(part)
    if any(g < 1 for g in part) or sum(part) != T:
        raise OracleError(f"partition {part} is not a composition of T={T}")
    out = []
    W = 0
    for g in part:
        lo = S * W
        W += g
        hi = min(S * W, ntiles)
        out.append((lo, hi))
    return out


def group_thresholds(partition, S: int, ntiles: int) -> list[int]:
    """|G_j| in tiles: the count at which group j's communication fires
    ("Once the j-th number reaches |G_j|")."""
    return [hi - lo for lo, hi in group_ranges(partition, S, ntiles)]


def group_of_position(partition, S: int, ntiles: int) -> np.ndarray:
    g = np.empty(ntiles, dtype=np.int64)
    for j, (lo, hi) in enumerate(group_ranges(partition, S, ntiles)):
        g[lo:hi] = j
    return g


@dataclass
class Plan:
    """Everything O1-O3 fix for one rank."""
    M: int
    N: int
    BM: int
    BN: int
    S: int
    order: np.ndarray
    partition: list
    Mt: int = 0
    Nt: int = 0
    T: int = 0
    ranges: list = field(default_factory=list)

    @property
    def ntiles(self) -> int:
        return self.Mt * self.Nt

    def tile_of_position(self, p: int) -> tuple[int, int]:
        return tile_coords(int(self.order[p]), self.Nt)


def make_plan(M, N, BM, BN, S, partition, order=None, swizzle=1) -> Plan:
    Mt, Nt = tile_grid(M, N, BM, BN)
    o = default_order(Mt, Nt, swizzle) if order is None else validate_order(order, Mt * Nt)
    T = num_waves(Mt * Nt, S)
    if partition is None:
        partition = [T]
    rg = group_ranges(partition, S, Mt * Nt)
    return Plan(M, N, BM, BN, S, o, [int(g) for g in partition], Mt, Nt, T, rg)
