"""Pins for oracle step O4 (fp64 GEMM) and the bf16 RNE model."""
import numpy as np
import torch

import synthetic
from oracle import numerics


def test_gemm_vs_brute_force():
    rng = np.random.default_rng(1)
    for _ in range(5):
        M, N, K = rng.integers(1, 7, size=3)
        A = torch.from_numpy(rng.standard_normal((M, K))).to(torch.bfloat16)
        Bt = torch.from_numpy(rng.standard_normal((N, K))).to(torch.bfloat16)
        C = numerics.gemm(A, Bt)
        Af, Bf = A.double().numpy(), Bt.double().numpy()
        for i in range(M):
            for j in range(N):
                s = 0.0
                for k in range(K):
                    s += Af[i, k] * Bf[j, k]
                assert abs(C[i, j] - s) <= 1e-12 * max(1.0, abs(s))


def test_gemm_exact_integer_regime_bound():
    A, Bt = synthetic.exact_inputs(64, 48, 512, seed=3, nnz_per_row=256)
    C = numerics.gemm(A, Bt)
    assert np.array_equal(C, np.rint(C))
    assert np.abs(C).max() <= 256
    # exactly representable in bf16
    assert np.array_equal(numerics.round_bf16(C), C)


def test_round_bf16_matches_torch_on_fp32_values():
    g = torch.Generator().manual_seed(0)
    x = torch.randn(200000, generator=g) * torch.exp(torch.randn(200000, generator=g) * 4)
    # include exact ties: bf16 value + half ulp
    base = torch.randn(1000, generator=g).to(torch.bfloat16).float()
    ulp = torch.ldexp(torch.ones_like(base), torch.frexp(base).exponent - 8)
    x = torch.cat([x, base + ulp / 2, base - ulp / 2])
    ref = x.to(torch.bfloat16).double().numpy()
    got = numerics.round_bf16(x.double().numpy())
    assert np.array_equal(got, ref)


def test_round_bf16_hand_ties():
    # 1 + 2^-8 is the midpoint between 1 and 1 + 2^-7 -> ties to even -> 1
    assert numerics.round_bf16(np.array([1 + 2.0 ** -8]))[0] == 1.0
    # 1 + 3*2^-8 is the midpoint between 1+2^-7 and 1+2^-6 -> even -> 1+2^-6
    assert numerics.round_bf16(np.array([1 + 3 * 2.0 ** -8]))[0] == 1 + 2.0 ** -6
    assert numerics.round_bf16(np.array([0.0]))[0] == 0.0
    assert numerics.round_bf16(np.array([-256.0]))[0] == -256.0
    assert numerics.round_bf16(np.array([257.0]))[0] == 256.0
