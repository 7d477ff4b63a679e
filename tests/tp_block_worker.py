"""The TP block (tools/tp_block.py, NEXT f4) on W ranks vs the oracle's TP
block (oracle/block.py), test infrastructure launched by
tests/test_gpu_graph.py in a subprocess: W = 1 with the library's NCCL
context, W = 2 with the loopback communicator (two in-process ranks on one
GPU, one host thread each).  Weights and inputs are drawn on the CPU from the
seeded generators; the library's output y and updated residual stream h of
every rank, overlapped and sequential, must be within TOL = 2^-6 (max |g - o| /
max(|o|, rms(o)), R11) of the oracle, which rounds to bf16 exactly
where the library stores bf16.  The tolerance is derived from that arithmetic:
a stored bf16 value may sit one ulp (2^-7 relative) from the oracle's when the
GPU's fp32 accumulation lands on the other side of a rounding boundary, and
the block adds two stored values before storing again (c + x, then y = h +
down), so two ulps: 2^-6 = 1.5625e-2 (measured: 7.8e-3 / 9.2e-3 at TP = 1,
1.3e-2 at TP = 2, where the AllReduce's bf16 sum is one more stored value).

usage: tp_block_worker.py W  -> prints "tp block W=<W>: OK" and exits 0.
"""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from oracle import block as ob  # noqa: E402
from tools.tp_block import Block, block_weights  # noqa: E402


TOL = 2.0 ** -6


def rel_err(g, o):
    rms = np.sqrt(np.mean(o * o))
    return float(np.max(np.abs(g - o) / np.maximum(np.abs(o), rms)))


def main(W):
    torch.cuda.set_device(0)
    T, H, I = 512, 1024, 2048
    if W == 1:
        ctxs = [fo.Context.create(0, 0, 1, fo.unique_id())]
        grp = None
    else:
        grp = fo.LoopbackGroup(0, W)
        ctxs = grp.contexts()
    weights = [block_weights(H, I, r, W, device="cpu") for r in range(W)]
    attn = [synthetic.normal_bf16((T, H // W), 1.0, 700 + r) for r in range(W)]
    x0 = synthetic.normal_bf16((T, H), 1.0, 8)
    want_y, want_h = ob.tp_block([a.double().numpy() for a in attn], x0.double().numpy(),
                                 [w[0].double().numpy() for w in weights], [w[1].double().numpy() for w in weights],
                                 [w[2].double().numpy() for w in weights], weights[0][3].double().numpy())
    blocks = [Block(ctxs[r], T, H, I, r, W, tuned=False, weights=weights[r]) for r in range(W)]
    for b in blocks:
        for p in (b.p_o, b.p_d, b.p_gu):     # nothing allocates while another rank's call is in flight
            p.prepare(sequential=True)
    attn_d = [a.cuda() for a in attn]
    streams = [torch.cuda.Stream() for _ in range(W)]
    pool = ThreadPoolExecutor(W)
    bad = []
    for ov in (True, False):
        xs = [x0.cuda() for _ in range(W)]
        ys = [None] * W
        torch.cuda.synchronize()

        def one(r):
            torch.cuda.set_device(0)
            with torch.cuda.stream(streams[r]):
                ys[r] = blocks[r].forward(attn_d[r], xs[r], overlapped=ov)
            streams[r].synchronize()
        for f in [pool.submit(one, r) for r in range(W)]:
            f.result()
        for r in range(W):
            ey = rel_err(ys[r].double().cpu().numpy(), want_y)
            eh = rel_err(xs[r].double().cpu().numpy(), want_h)
            print(f"W={W} rank {r} {'overlapped' if ov else 'sequential'}: y {ey:.3e}  h {eh:.3e}", flush=True)
            if not (ey <= TOL and eh <= TOL):
                bad.append((r, ov, ey, eh))
    for c in ctxs:
        c.close()
    if grp is not None:
        grp.close()
    print(f"tp block W={W}: " + ("OK" if not bad else f"FAILED {bad}"), flush=True)
    return 0 if not bad else 1


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1])))
