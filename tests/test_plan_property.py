"""Property-based parity of the C++ plan (host library) against the oracle:
hypothesis draws tile shapes, grids, wave widths, partitions, explicit or
default orders, collectives and world sizes; every send / receive map must
equal the oracle's, bit-exactly (CPU only)."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import plan as op
from oracle import reorder as orr

fo = pytest.importorskip("paper_2504_19519_b200")


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2504_19519_b200 import build

    build.build()


@st.composite
def plans(draw):
    BM = draw(st.sampled_from([128, 256]))
    BN = draw(st.sampled_from([64, 128, 256]))
    Mt = draw(st.integers(1, 4))
    Nt = draw(st.integers(1, 4))
    tiles = Mt * Nt
    S = draw(st.integers(1, tiles + 2))
    T = -(-tiles // S)
    cuts = draw(st.lists(st.booleans(), min_size=T - 1, max_size=T - 1))
    part, run = [], 0
    for w in range(T):
        run += 1
        if w == T - 1 or cuts[w]:
            part.append(run)
            run = 0
    explicit = draw(st.booleans())
    order = draw(st.permutations(list(range(tiles)))) if explicit else None
    swz = draw(st.integers(1, 5))
    coll = draw(st.sampled_from(["allreduce", "reducescatter"]))
    world = draw(st.sampled_from([1, 2, 4, 8])) if coll == "reducescatter" else 1
    layout = draw(st.sampled_from(["slot", "auto"]))
    return dict(BM=BM, BN=BN, M=Mt * BM, N=Nt * BN, S=S, part=part, order=order, swz=swz, coll=coll,
                world=world, layout=layout)


@settings(max_examples=150, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(c=plans())
def test_plan_maps_match_oracle(c):
    o = op.make_plan(c["M"], c["N"], c["BM"], c["BN"], c["S"], c["part"], order=c["order"], swizzle=c["swz"])
    rank = c["world"] - 1
    pl = fo.Plan(coll=c["coll"], m=c["M"], n=c["N"], k=64, tile_m=c["BM"], tile_n=c["BN"], workers=c["S"],
                 tile_order=c["order"], swizzle=c["swz"], group_waves=c["part"], ar_layout=c["layout"],
                 rank=rank, world=c["world"])
    assert pl.export_order().tolist() == o.order.tolist()
    Y = np.arange(c["M"] * c["N"], dtype=float).reshape(c["M"], c["N"])
    if c["coll"] == "allreduce":
        lay = "rowband" if pl.info["ar_layout"] == 1 else "slot"
        assert (lay == "rowband") == (c["layout"] == "auto" and orr.ar_rowband_ok(o))
        buf = orr.ar_pre(Y, o, lay)
        post = orr.ar_post(np.arange(c["M"] * c["N"], dtype=float), o, lay)
        ranges = orr.group_elem_ranges(o, lay)
    else:
        lay = "rowband" if pl.info["ar_layout"] == 1 else "slot"
        assert (lay == "rowband") == (c["layout"] == "auto" and orr.rs_rowband_ok(o))
        buf = orr.rs_pre(Y, o, c["world"], lay)
        post = orr.rs_post(np.arange(c["M"] * c["N"] // c["world"], dtype=float), o, c["world"], lay)
        ranges = orr.group_elem_ranges(o, lay)
    inv = np.empty(buf.size, np.int64)
    inv[buf.astype(np.int64)] = np.arange(buf.size)
    assert np.array_equal(pl.export_send_map(), inv)
    assert np.array_equal(pl.export_recv_map(), post.reshape(-1).astype(np.int64))
    for j, ((lo, hi), (elo, ehi)) in enumerate(zip(o.ranges, ranges)):
        assert pl.group(j) == (lo, hi, elo, ehi)
