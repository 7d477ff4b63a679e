"""One-wave GEMM shapes (M = 1024: 64 tiles of 256x256 on 64 CTA pairs) — the
plain persistent grid vs TMA multicast across clusters of two pairs
(FO_OPT_MULTICAST) vs K-snake off vs cuBLAS (dev probe; interleaved, L2
flushed, stream pre-loaded, medians of 15)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2504_19519_b200 as fo  # noqa: E402
import synthetic  # noqa: E402
from tools.probes.suffix_probe import timeit_many  # noqa: E402


def main():
    torch.cuda.set_device(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for (M, N, K) in [(1024, 4096, 4096), (1024, 4096, 14336), (1024, 8192, 8192), (2048, 4096, 4096),
                      (4096, 4096, 4096)]:
        A, Bt = synthetic.float_inputs(M, N, K, seed=1, device="cuda")
        C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        tiles = (M // 256) * (N // 256)
        S = min(64, tiles) if tiles <= 74 else 64
        v = {}
        for name, opts in (("plain", {}), ("multicast", {"multicast": 1}), ("no-ksnake", {"k_snake": 0}),
                           ("swz1", None)):
            p = fo.Plan(coll="nocomm", m=M, n=N, k=K, tile_m=256, tile_n=256, workers=S,
                        swizzle=1 if opts is None else 0)
            for k_, val in (opts or {}).items():
                p.set_option(k_, val)
            v[name] = (lambda p=p: fo.gemm_stage(p, A, Bt, C))
            if name == "multicast":
                v[name + f"(cluster={p.gemm_cluster()})"] = v.pop(name)
        v["cuBLAS"] = lambda: torch.matmul(A, Bt.t(), out=C)
        t = timeit_many(list(v.values()), flush)
        fl = 2.0 * M * N * K
        print(f"{M}x{N}x{K} ({tiles} tiles, S={S}): " + "  ".join(
            f"{k} {x:.1f} us ({fl / x / 1e6:.0f})" for k, x in zip(v, t)), flush=True)
        del A, Bt, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
