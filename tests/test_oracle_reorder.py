"""Pins for oracle steps O5/O7 (pre/post-communication reordering) and O9."""
import json
import os

import numpy as np
import pytest

import synthetic
from oracle import collectives as oc
from oracle import pipeline as opl
from oracle import plan as op
from oracle import reorder as orr

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reorder.json")))


def _rand_plan(rng, BMs=(1, 2, 4), n=1):
    BM = int(rng.choice(BMs)) * n
    BN = int(rng.integers(1, 4))
    Mt, Nt = int(rng.integers(1, 5)), int(rng.integers(1, 5))
    ntiles = Mt * Nt
    S = int(rng.integers(1, ntiles + 1))
    T = op.num_waves(ntiles, S)
    part = synthetic.random_partition(T, int(rng.integers(1 << 30)))
    order = synthetic.random_order(ntiles, int(rng.integers(1 << 30)))
    return op.make_plan(Mt * BM, Nt * BN, BM, BN, S, part, order=order)


def test_ar_roundtrip_and_bijection():
    """post(pre(X)) == X bit-exactly; pre is a bijection."""
    rng = np.random.default_rng(0)
    for _ in range(300):
        pl = _rand_plan(rng)
        X = rng.standard_normal((pl.M, pl.N))
        buf = orr.ar_pre(X, pl)
        assert np.array_equal(orr.ar_post(buf, pl), X)
        idx = orr.ar_pre(np.arange(pl.M * pl.N, dtype=float).reshape(pl.M, pl.N), pl)
        assert np.array_equal(np.sort(idx), np.arange(pl.M * pl.N))


def test_ar_group_contiguity_and_monotonicity():
    """Every element of group j sits inside group j's range, ranges ordered
    (SPEC.md:150-152)."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        pl = _rand_plan(rng)
        idx = orr.ar_pre(np.arange(pl.M * pl.N, dtype=float).reshape(pl.M, pl.N), pl).astype(int)
        gop = op.group_of_position(pl.partition, pl.S, pl.ntiles)
        pos_of_tile = {int(t): p for p, t in enumerate(pl.order)}
        for (lo, hi), j in zip(orr.group_elem_ranges(pl), range(len(pl.ranges))):
            for e in idx[lo:hi]:
                r, c = divmod(int(e), pl.N)
                t = (r // pl.BM) * pl.Nt + c // pl.BN
                assert gop[pos_of_tile[t]] == j
        starts = [lo for lo, _ in orr.group_elem_ranges(pl)]
        assert starts == sorted(starts)


def test_ar_rowband_is_identity_layout():
    pl = op.make_plan(8, 6, 2, 2, 6, [1, 1], swizzle=1)   # 4x3 tiles, waves of 2 tile-rows
    X = np.arange(48.0).reshape(8, 6)
    assert orr.ar_rowband_ok(pl)
    assert np.array_equal(orr.ar_pre(X, pl, "rowband"), X.reshape(-1))
    assert orr.group_elem_ranges(pl, "rowband") == [(0, 24), (24, 48)]
    bad = op.make_plan(8, 6, 2, 2, 4, [1, 1, 1], swizzle=1)  # group boundary mid tile-row
    assert not orr.ar_rowband_ok(bad)
    with pytest.raises(op.OracleError):
        orr.ar_pre(X, bad, "rowband")
    # swizzled order whose groups are whole row-panels: still a row band per group
    sw = op.make_plan(8, 6, 2, 2, 6, [1, 1], swizzle=2)   # panel of 2 tile-rows = 6 tiles = 1 wave
    assert orr.ar_rowband_ok(sw)
    # a group made of two non-adjacent tile-rows is not a band
    nb = op.make_plan(8, 6, 2, 2, 6, [1, 1], order=[0, 1, 2, 6, 7, 8, 3, 4, 5, 9, 10, 11])
    assert not orr.ar_rowband_ok(nb)


def test_ar_rowband_roundtrip_random_bands():
    """Rowband AR pipeline == plain definition for random band partitions with
    random within-band orders and bands in arbitrary order."""
    from oracle import pipeline as opl
    rng = np.random.default_rng(9)
    for _ in range(50):
        Mt, Nt, BM, BN = int(rng.integers(1, 6)), int(rng.integers(1, 4)), 2, 2
        S = Nt * int(rng.integers(1, 3))          # wave = whole tile-rows
        rows_per_wave = S // Nt
        T = -(-Mt // rows_per_wave)
        part = synthetic.random_partition(T, int(rng.integers(1 << 20)))
        # assign bands to groups in a random order of bands
        band_rows = list(range(Mt))
        order = []
        for r in band_rows:
            order += list(rng.permutation(np.arange(r * Nt, (r + 1) * Nt)))
        pl = op.make_plan(Mt * BM, Nt * BN, BM, BN, S, part, order=order)
        assert orr.ar_rowband_ok(pl)
        As = [rng.integers(-3, 4, size=(Mt * BM, 3)).astype(float) for _ in range(2)]
        Bts = [rng.integers(-3, 4, size=(Nt * BN, 3)).astype(float) for _ in range(2)]
        res = opl.run_allreduce(As, Bts, pl, layout="rowband")
        assert np.array_equal(res["out"][0], opl.plain_allreduce(As, Bts)[0])


def test_rs_worked_example_g6():
    c = GOLD["rs"][0]
    pl = op.make_plan(c["M"], c["N"], c["BM"], c["BN"], c["S"], c["partition"])
    Y = np.repeat(np.arange(c["M"], dtype=float)[:, None], c["N"], axis=1)  # value = row id
    buf = orr.rs_pre(Y, pl, c["n"])
    assert buf.reshape(-1, c["N"])[:, 0].astype(int).tolist() == c["buffer_rows"]
    for k in range(c["n"]):
        chunk = orr.rs_chunk(buf, pl, c["n"], 0, k)
        assert chunk.reshape(-1, c["N"])[:, 0].astype(int).tolist() == c["rank_rows"][k]
        assert opl.rs_rows_of_rank(c["M"], c["BM"], c["n"], k).tolist() == c["rank_rows"][k]


def test_row_exchange_spec_example():
    c = GOLD["rs"][1]
    gathered = np.array(c["gathered"], dtype=float)[:, None]
    assert opl.row_exchange(gathered, c["BM"], c["n"])[:, 0].astype(int).tolist() == list(range(c["M"]))


def test_rs_rows_complete_on_one_rank():
    """after RS each row resides entirely on one GPU."""
    rng = np.random.default_rng(2)
    for n in (1, 2, 3, 4):
        for _ in range(40):
            pl = _rand_plan(rng, n=n)
            M, N = pl.M, pl.N
            Y = (np.arange(M)[:, None] * 1000 + np.arange(N)[None, :]).astype(float)
            bufs = [orr.rs_pre(Y, pl, n) for _ in range(n)]
            recv = oc.reduce_scatter_groups(bufs, orr.group_elem_ranges(pl))
            covered = np.zeros(M, int)
            for k in range(n):
                out = orr.rs_post(recv[k], pl, n)
                for l in range(M // n):
                    g = orr.rs_local_to_global_row(l, pl.BM, pl.BM // n, k)
                    assert np.array_equal(out[l], n * Y[g])
                    covered[g] += 1
            assert (covered == 1).all()


def test_rs_pre_inverse():
    """O9 for RS with n = 1 (identity collective): post(pre(X)) == X."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        pl = _rand_plan(rng)
        X = rng.standard_normal((pl.M, pl.N))
        buf = orr.rs_pre(X, pl, 1)
        assert np.array_equal(orr.rs_post(buf, pl, 1), X)
        idx = orr.rs_pre(np.arange(pl.M * pl.N, dtype=float).reshape(pl.M, pl.N), pl, 1)
        assert np.array_equal(np.sort(idx), np.arange(pl.M * pl.N))


def test_rs_indivisible_rejected():
    pl = op.make_plan(6, 2, 3, 2, 1, None)
    with pytest.raises(op.OracleError):
        orr.rs_pre(np.zeros((6, 2)), pl, 2)


def test_a2a_worked_example_g7():
    c = GOLD["a2a"][0]
    pl = op.make_plan(c["M"], c["N"], c["BM"], c["BN"], c["S"], c["partition"])
    Y = np.arange(c["M"] * c["N"], dtype=float).reshape(c["M"], c["N"])
    s = orr.a2a_pre(Y, pl, c["row_dst"], c["n"])
    for d in range(c["n"]):
        assert [list(m) for m in s.meta[d]] == c["pool_meta"][d]
        assert [list(r) for r in s.ranges[d]] == c["pool_ranges"][d]
        for (row, j), v in zip(s.meta[d], s.pools[d]):
            assert np.array_equal(v, Y[row, j * c["BN"]:(j + 1) * c["BN"]])
    assert np.flatnonzero(np.array(c["row_dst"]) == 0).tolist() == c["rank0_rows_from_self"]


def test_a2a_identity_routing_roundtrip():
    """A2A with every row routed to the only rank is a permutation + inverse."""
    rng = np.random.default_rng(4)
    for _ in range(60):
        pl = _rand_plan(rng)
        X = rng.standard_normal((pl.M, pl.N))
        s = orr.a2a_pre(X, pl, np.zeros(pl.M, int), 1)
        recv = oc.alltoall_groups([s], len(pl.ranges))
        out = orr.a2a_post(recv[0], [s.meta[0]], [np.zeros(pl.M, int)], 0, pl.N, pl.BN)
        assert np.array_equal(out, X)


def test_a2a_errors():
    pl = op.make_plan(4, 4, 2, 2, 2, None)
    with pytest.raises(op.OracleError):
        orr.a2a_pre(np.zeros((4, 4)), pl, [0, 1, 2], 2)
    with pytest.raises(op.OracleError):
        orr.a2a_pre(np.zeros((4, 4)), pl, [0, 1, 2, 0], 2)


# ---------------------------------------------------------------- RS rowband (R40)
def _band_plan(rng, n):
    """A plan whose groups are ascending bands of complete tile-rows (random
    tile order inside each band, random band sizes)."""
    BM = int(rng.choice((1, 2))) * n
    BN = int(rng.integers(1, 4))
    Mt, Nt = int(rng.integers(1, 6)), int(rng.integers(1, 4))
    rows_per_wave = int(rng.integers(1, Mt + 1))
    S = rows_per_wave * Nt
    T = -(-Mt // rows_per_wave)
    part = synthetic.random_partition(T, int(rng.integers(1 << 20)))
    order = []
    for r in range(Mt):
        order += [int(t) for t in rng.permutation(np.arange(r * Nt, (r + 1) * Nt))]
    # tile-rows in ascending order, tiles of one tile-row shuffled among the band
    return op.make_plan(Mt * BM, Nt * BN, BM, BN, S, part, order=order)


def test_rs_rowband_hand_example():
    """4x4 output, 2x2 tiles, n = 2 (h = 1), one group of both tile-rows:
    chunk 0 = the k=0 subtile rows of tile-rows 0 and 1 = global rows 0, 2;
    chunk 1 = rows 1, 3 (worked by hand from PAPER.md:390: the k-th subtile
    of every tile goes to GPU k).  Rank 0 then holds R_0 = {0, 2}."""
    pl = op.make_plan(4, 4, 2, 2, 4, [1], swizzle=1)
    Y = np.repeat(np.arange(4, dtype=float)[:, None], 4, axis=1)  # value = row id
    assert orr.rs_rowband_ok(pl)
    buf = orr.rs_pre(Y, pl, 2, "rowband")
    assert buf.reshape(4, 4)[:, 0].astype(int).tolist() == [0, 2, 1, 3]
    assert orr.rs_chunk(buf, pl, 2, 0, 0, "rowband").reshape(-1, 4)[:, 0].tolist() == [0, 2]
    assert orr.rs_chunk(buf, pl, 2, 0, 1, "rowband").reshape(-1, 4)[:, 0].tolist() == [1, 3]
    # two groups of one tile-row each: every chunk is one row, in row order
    pl2 = op.make_plan(4, 4, 2, 2, 2, [1, 1], swizzle=1)
    buf2 = orr.rs_pre(Y, pl2, 2, "rowband")
    assert buf2.reshape(4, 4)[:, 0].astype(int).tolist() == [0, 1, 2, 3]


def test_rs_rowband_legality():
    """Bands must be complete tile-rows AND ascending in group order."""
    # raster, waves = whole tile-rows: legal
    assert orr.rs_rowband_ok(op.make_plan(8, 4, 2, 2, 2, [1, 1, 1, 1], swizzle=1))
    # tile-row 1 before tile-row 0: bands exist but descend
    pl = op.make_plan(4, 4, 2, 2, 2, [1, 1], order=[2, 3, 0, 1])
    assert orr.ar_rowband_ok(pl) and not orr.rs_rowband_ok(pl)
    with pytest.raises(op.OracleError):
        orr.rs_pre(np.zeros((4, 4)), pl, 2, "rowband")
    # column-major inside a 2-row panel with single-wave groups of 2 tiles: not bands
    assert not orr.rs_rowband_ok(op.make_plan(4, 4, 2, 2, 2, [1, 1], swizzle=2))


def test_rs_rowband_equals_definition_bruteforce():
    """Overlapped RS in the rowband layout == plain RS (rows R_k of the sum),
    on integer data, for random band plans at n = 1..4; the layout is a
    bijection and its receive buffer is the output itself (row-major)."""
    rng = np.random.default_rng(40)
    for n in (1, 2, 3, 4):
        for _ in range(40):
            pl = _band_plan(rng, n)
            assert orr.rs_rowband_ok(pl)
            K = 3
            As = [rng.integers(-3, 4, size=(pl.M, K)).astype(float) for _ in range(n)]
            Bts = [rng.integers(-3, 4, size=(pl.N, K)).astype(float) for _ in range(n)]
            res = opl.run_reducescatter(As, Bts, pl, layout="rowband")
            plain = opl.plain_reducescatter(As, Bts, pl.BM)
            for k in range(n):
                assert np.array_equal(res["out"][k], plain[k])
                assert np.array_equal(res["recv"][k], res["out"][k].reshape(-1))
            idx = orr.rs_pre(np.arange(pl.M * pl.N, dtype=float).reshape(pl.M, pl.N), pl, n, "rowband")
            assert np.array_equal(np.sort(idx), np.arange(pl.M * pl.N))
            # same output as the paper's subtile (slot) layout
            slot = opl.run_reducescatter(As, Bts, pl)
            for k in range(n):
                assert np.array_equal(slot["out"][k], res["out"][k])


# ---------------------------------------------------------------- A2A rowband (R41)
def test_a2a_rowband_hand_example():
    """4x4 output of 2x2 tiles, row_dst = [1, 0, 1, 1], raster, one tile-row
    per group.  Worked by hand: the paper's layout (subtokens in
    execution order p, then row) fills pool 1 with (0,0),(0,1),(2,0),(3,0),
    (2,1),(3,1); the rowband layout keeps rows whole: (0,0),(0,1),(2,0),(2,1),
    (3,0),(3,1); pool 0 is (1,0),(1,1) in both."""
    pl = op.make_plan(4, 4, 2, 2, 2, [1, 1], swizzle=1)
    Y = np.arange(16, dtype=float).reshape(4, 4)
    rd = [1, 0, 1, 1]
    slot = orr.a2a_pre(Y, pl, rd, 2)
    band = orr.a2a_pre(Y, pl, rd, 2, "rowband")
    assert slot.meta[1] == [(0, 0), (0, 1), (2, 0), (3, 0), (2, 1), (3, 1)]
    assert band.meta[1] == [(0, 0), (0, 1), (2, 0), (2, 1), (3, 0), (3, 1)]
    assert band.meta[0] == slot.meta[0] == [(1, 0), (1, 1)]
    assert band.ranges[1] == [(0, 2), (2, 6)] and band.ranges[0] == [(0, 2), (2, 2)]
    assert np.array_equal(band.pools[1].reshape(-1), Y[[0, 2, 3]].reshape(-1))


def test_a2a_rowband_equals_definition_bruteforce():
    """Per-group A2A in the rowband layout == the plain all-to-all-v, for
    imbalanced sources with random routing at n = 1..4; and what a receiver
    gets from one source in one group is a run of consecutive complete output
    rows (so it can be received straight into the output)."""
    rng = np.random.default_rng(41)
    for n in (1, 2, 3, 4):
        for _ in range(25):
            BM, BN, Nt = int(rng.choice((1, 2, 3))), int(rng.integers(1, 3)), int(rng.integers(1, 3))
            P = int(rng.integers(1, 3))
            plans, rds, As, Bts = [], [], [], []
            for _s in range(n):
                Mt = int(rng.integers(P, P + 3))
                plans.append(op.make_plan(Mt * BM, Nt * BN, BM, BN, Nt, [1] * (P - 1) + [Mt - P + 1], swizzle=1))
                rds.append(rng.integers(0, n, size=Mt * BM))
                As.append(rng.integers(-3, 4, size=(Mt * BM, 2)).astype(float))
                Bts.append(rng.integers(-3, 4, size=(Nt * BN, 2)).astype(float))
            assert orr.a2a_rowband_ok(plans)
            res = opl.run_alltoall(As, Bts, plans, rds, layout="rowband")
            plain = opl.plain_alltoall(As, Bts, rds)
            for d in range(n):
                assert np.array_equal(res["out"][d], plain[d])
            for s_ in range(n):
                snd = res["send"][s_]
                for d in range(n):
                    rows_to_d = list(np.flatnonzero(np.asarray(rds[s_]) == d))
                    for (a, b) in snd.ranges[d]:
                        meta = snd.meta[d][a:b]
                        assert len(meta) % Nt == 0
                        rows = [meta[i][0] for i in range(0, len(meta), Nt)]
                        assert all(meta[i] == (rows[i // Nt], i % Nt) for i in range(len(meta)))
                        if rows:
                            k0 = rows_to_d.index(rows[0])
                            assert rows == rows_to_d[k0:k0 + len(rows)]
