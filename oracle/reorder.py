"""Oracle steps O5 (pre-communication reordering) and O7 (post-communication
reordering) for AllReduce, ReduceScatter and All-to-All.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:385-386: "the reordered output is first reshaped into a column of tiles
(row major) before communication.  For the inter-tile data contiguity, the tile
indices are reordered based on their execution order".

  AR: unit = tile.  Tile at execution position p goes to slot p
      (reading R2: slot = execution position), each slot BM*BN
      contiguous elements, row-major inside the slot.
      Layout "rowband" (H11a): when the tiles of every group are
      exactly the complete tile-rows of one contiguous band [r0, r1) (any
      execution order inside the group), the slot layout is replaced by the
      identity (the buffer IS row-major C) and group j communicates its row
      band [r0*BM*N, r1*BM*N).  Both layouts are valid AR reorderings
      (only a consistent order across GPUs is required).
  RS: unit = subtile of h = BM/n rows.  Inside group j (positions
      [ps, pe), G = pe - ps), chunk k (the part ReduceScatter delivers to rank k)
      holds the k-th subtile of every tile of the group, tiles in execution
      order:  buf[ps*BM*BN + k*G*h*BN + q*h*BN + a'*BN + b]
                 = Y[i*BM + k*h + a', j*BN + b],   q = p - ps.
      Layout "rowband" (R40): when the groups are the bands of whole
      tile-rows [r0, r1) in ascending order (band j starts where band j-1
      ends), the unit is still the k-th subtile ("the k-th subtile
      within a tile always resides on the k-th GPU"), but chunk k of band j
      holds the k-th subtiles as complete rows, tile-row by tile-row
      (B = r1 - r0):
              buf[r0*BM*N + k*B*h*N + ((i - r0)*h + a')*N + c]
                 = Y[i*BM + k*h + a', c],   i in [r0, r1)
      so rank k receives its block-cyclic rows R_k already in output order.
  A2A: unit = subtoken (one row of one tile, BN elements).  One
      memory pool per destination rank; subtokens are appended in execution
      order (p ascending, then row inside the tile ascending).  Group j's
      subtokens form one contiguous range of every pool.
      Layout "rowband" (R41): when every source's groups are
      ascending bands of whole tile-rows, group j's subtokens are appended
      row by row (source row ascending, then tile-column ascending), i.e.
      pool d holds complete rows in source-row order; the part of group j a
      receiver gets from source s is then a run of consecutive output rows.

Pins (tests/test_oracle_reorder.py): post(pre(X)) == X bit-exactly
("the output in (d) is the same as (a)"); every element lands in
exactly one buffer position (bijection); group ranges contiguous and ordered
(monotonicity); RS: each row complete on exactly one rank;
SURVEY g5/g6/g7 worked cases and SPEC.md:145's gathered row order
[0,1,4,5,2,3,6,7].
"""
from __future__ import annotations

import numpy as np

from .plan import OracleError, Plan


# =========================================================== AllReduce
def rowband_of_group(plan: Plan, lo: int, hi: int):
    """(r0, r1) if the tiles at positions [lo, hi) are exactly the complete
    tile-rows r0..r1-1, else None."""
    tiles = sorted(int(t) for t in plan.order[lo:hi])
    if not tiles or len(tiles) % plan.Nt:
        return None
    r0 = tiles[0] // plan.Nt
    r1 = r0 + len(tiles) // plan.Nt
    if tiles != list(range(r0 * plan.Nt, r1 * plan.Nt)):
        return None
    return r0, r1


def rs_rowband_ok(plan: Plan) -> bool:
    """ReduceScatter rowband layout: every group is a band of complete
    tile-rows and the bands follow each other top to bottom in group order
    (the receive buffer concatenates the groups' chunks in group order)."""
    nxt = 0
    for lo, hi in plan.ranges:
        if lo == hi and plan.ntiles == 0:
            continue   # an All-to-All source with no rows: empty groups, empty bands (R45)
        band = rowband_of_group(plan, lo, hi)
        if band is None or band[0] != nxt:
            return False
        nxt = band[1]
    return True


def ar_rowband_ok(plan: Plan) -> bool:
    """Identity layout is valid iff every group's tiles form one band of
    complete, contiguous tile-rows (so each group is a row band of C)."""
    return all(rowband_of_group(plan, lo, hi) is not None for lo, hi in plan.ranges)


def group_elem_ranges(plan: Plan, layout: str = "slot") -> list[tuple[int, int]]:
    """Element range [lo, hi) of each group in the AR / RS send buffer."""
    if layout == "rowband":
        band = [rowband_of_group(plan, lo, hi) for lo, hi in plan.ranges]
        return [(r0 * plan.BM * plan.N, r1 * plan.BM * plan.N) for r0, r1 in band]
    t = plan.BM * plan.BN
    return [(lo * t, hi * t) for lo, hi in plan.ranges]


def ar_pre(Y: np.ndarray, plan: Plan, layout: str = "slot") -> np.ndarray:
    """O5 for AllReduce: Y [M, N] -> flat buffer of M*N elements."""
    BM, BN = plan.BM, plan.BN
    if layout == "rowband":
        if not ar_rowband_ok(plan):
            raise OracleError("rowband layout needs every group to be a band of complete tile-rows")
        return Y.reshape(-1).copy()
    buf = np.empty(plan.M * plan.N, dtype=Y.dtype)
    for p in range(plan.ntiles):
        i, j = plan.tile_of_position(p)
        buf[p * BM * BN:(p + 1) * BM * BN] = Y[i * BM:(i + 1) * BM, j * BN:(j + 1) * BN].reshape(-1)
    return buf


def ar_post(buf: np.ndarray, plan: Plan, layout: str = "slot") -> np.ndarray:
    """O7 for AllReduce: the inverse of ar_pre."""
    BM, BN = plan.BM, plan.BN
    if layout == "rowband":
        return buf.reshape(plan.M, plan.N).copy()
    Y = np.empty((plan.M, plan.N), dtype=buf.dtype)
    for p in range(plan.ntiles):
        i, j = plan.tile_of_position(p)
        Y[i * BM:(i + 1) * BM, j * BN:(j + 1) * BN] = buf[p * BM * BN:(p + 1) * BM * BN].reshape(BM, BN)
    return Y


# =========================================================== ReduceScatter
def rs_subtile_rows(plan: Plan, n: int) -> int:
    if plan.BM % n:
        raise OracleError(f"tile_m={plan.BM} not divisible by world size {n}")
    return plan.BM // n


def rs_pre(Y: np.ndarray, plan: Plan, n: int, layout: str = "slot") -> np.ndarray:
    """O5 for ReduceScatter (formulas in the module header)."""
    BM, BN = plan.BM, plan.BN
    h = rs_subtile_rows(plan, n)
    buf = np.empty(plan.M * plan.N, dtype=Y.dtype)
    if layout == "rowband":
        if not rs_rowband_ok(plan):
            raise OracleError("RS rowband layout needs the groups to be ascending bands of complete tile-rows")
        N = plan.N
        for lo, hi in plan.ranges:
            r0, r1 = rowband_of_group(plan, lo, hi)
            B = r1 - r0
            for k in range(n):
                for i in range(r0, r1):
                    off = r0 * BM * N + k * B * h * N + (i - r0) * h * N
                    buf[off:off + h * N] = Y[i * BM + k * h:i * BM + (k + 1) * h, :].reshape(-1)
        return buf
    for ps, pe in plan.ranges:
        G = pe - ps
        for p in range(ps, pe):
            q = p - ps
            i, j = plan.tile_of_position(p)
            for k in range(n):
                off = ps * BM * BN + k * G * h * BN + q * h * BN
                sub = Y[i * BM + k * h:i * BM + (k + 1) * h, j * BN:(j + 1) * BN]
                buf[off:off + h * BN] = sub.reshape(-1)
    return buf


def rs_chunk(buf: np.ndarray, plan: Plan, n: int, group: int, k: int, layout: str = "slot") -> np.ndarray:
    """Chunk k of group `group`: what ReduceScatter on the group range delivers to rank k."""
    BM, BN = plan.BM, plan.BN
    h = rs_subtile_rows(plan, n)
    ps, pe = plan.ranges[group]
    if layout == "rowband":
        r0, r1 = rowband_of_group(plan, ps, pe)
        off = r0 * BM * plan.N + k * (r1 - r0) * h * plan.N
        return buf[off:off + (r1 - r0) * h * plan.N]
    G = pe - ps
    off = ps * BM * BN + k * G * h * BN
    return buf[off:off + G * h * BN]


def rs_local_to_global_row(l: int, BM: int, h: int, k: int) -> int:
    """Rank k's local output row l holds global row floor(l/h)*BM + k*h + (l mod h)
    (block-cyclic rows R_k, SURVEY.md §8(b) output contract)."""
    return (l // h) * BM + k * h + (l % h)


def rs_post(recv: np.ndarray, plan: Plan, n: int, layout: str = "slot") -> np.ndarray:
    """O7 for ReduceScatter on one rank: the received buffer (group chunks
    concatenated in group order, each G*h*BN elements) -> local [M/n, N] rows
    in block-cyclic order (local row i*h + a' <- tile-row i, subtile row a').
    Rowband: band j's chunk holds local rows [r0*h, r1*h) in order."""
    BM, BN = plan.BM, plan.BN
    h = rs_subtile_rows(plan, n)
    out = np.empty((plan.M // n, plan.N), dtype=recv.dtype)
    if layout == "rowband":
        off = 0
        for lo, hi in plan.ranges:
            r0, r1 = rowband_of_group(plan, lo, hi)
            sz = (r1 - r0) * h * plan.N
            out[r0 * h:r1 * h, :] = recv[off:off + sz].reshape((r1 - r0) * h, plan.N)
            off += sz
        return out
    for ps, pe in plan.ranges:
        for p in range(ps, pe):
            q = p - ps
            i, j = plan.tile_of_position(p)
            off = ps * h * BN + q * h * BN
            out[i * h:(i + 1) * h, j * BN:(j + 1) * BN] = recv[off:off + h * BN].reshape(h, BN)
    return out


# =========================================================== All-to-All
class A2ASend:
    """Per-source pools: pools[d] is an array [cnt_d, BN]; meta[d] the list of
    (row, tile_col) of each subtoken; ranges[d][j] = (start, end) subtoken range
    of group j in pool d."""

    def __init__(self, n: int, P: int):
        self.pools = [[] for _ in range(n)]
        self.meta = [[] for _ in range(n)]
        self.ranges = [[None] * P for _ in range(n)]


def a2a_rowband_ok(plans) -> bool:
    """A2A rowband: every source's groups are ascending bands of complete tile-rows."""
    return all(rs_rowband_ok(pl) for pl in plans)


def a2a_pre(Y: np.ndarray, plan: Plan, row_dst, n: int, layout: str = "slot") -> A2ASend:
    """O5 for All-to-All (module header)."""
    BM, BN = plan.BM, plan.BN
    row_dst = np.asarray(row_dst).reshape(-1)
    if row_dst.size != plan.M:
        raise OracleError("row_dst must give a destination for every output row")
    if row_dst.size and (row_dst.min() < 0 or row_dst.max() >= n):
        raise OracleError("row_dst out of range")
    P = len(plan.ranges)
    s = A2ASend(n, P)
    if layout == "rowband" and not rs_rowband_ok(plan):
        raise OracleError("A2A rowband layout needs ascending bands of complete tile-rows as groups")
    for gj, (ps, pe) in enumerate(plan.ranges):
        start = [len(s.pools[d]) for d in range(n)]
        if layout == "rowband":
            r0, r1 = rowband_of_group(plan, ps, pe) if pe > ps else (0, 0)
            for row in range(r0 * BM, r1 * BM):
                d = int(row_dst[row])
                for j in range(plan.Nt):
                    s.pools[d].append(Y[row, j * BN:(j + 1) * BN].copy())
                    s.meta[d].append((row, j))
            for d in range(n):
                s.ranges[d][gj] = (start[d], len(s.pools[d]))
            continue
        for p in range(ps, pe):
            i, j = plan.tile_of_position(p)
            for a in range(BM):
                row = i * BM + a
                d = int(row_dst[row])
                s.pools[d].append(Y[row, j * BN:(j + 1) * BN].copy())
                s.meta[d].append((row, j))
        for d in range(n):
            s.ranges[d][gj] = (start[d], len(s.pools[d]))
    for d in range(n):
        s.pools[d] = (np.array(s.pools[d]).reshape(-1, BN) if s.pools[d]
                      else np.zeros((0, BN), dtype=Y.dtype))
    return s


def a2a_post(recv_parts, sources_meta, sources_row_dst, me: int, N: int, BN: int) -> np.ndarray:
    """O7 for All-to-All on rank `me`.

    recv_parts: list over (group j, source s) in receive order of
    (s, subtoken_array) as produced by collectives.alltoall.
    sources_meta[s]: the (row, tile_col) list of pool s->me (source order).
    Output: rows grouped by source ascending; within a source, ascending
    source row (standard all-to-all-v order)."""
    n = len(sources_row_dst)
    rows_to_me = [np.flatnonzero(np.asarray(sources_row_dst[s]) == me) for s in range(n)]
    base = np.concatenate([[0], np.cumsum([len(r) for r in rows_to_me])]).astype(np.int64)
    rank_of = [{int(r): idx for idx, r in enumerate(rows_to_me[s])} for s in range(n)]
    out = np.zeros((int(base[-1]), N))
    consumed = [0] * n
    for s, chunk in recv_parts:
        for v in chunk:
            row, j = sources_meta[s][consumed[s]]
            consumed[s] += 1
            out[base[s] + rank_of[s][row], j * BN:(j + 1) * BN] = v
    return out
