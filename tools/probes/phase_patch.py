"""Make an instrumented copy of the package for tools/probes/phase_probe.py
(dev probe): copies paper_2504_19519_b200/, synthetic/, include/ and
__graft_entry__.py into DEST and patches the GEMM kernel with %globaltimer
stamps written after the per-tile area of the debug buffer (slot i of CTA b
at tile_ts[tiles + 16 b + i]).  The shipped kernel has no stamps.

    python tools/probes/phase_patch.py tools/probes/phase && (cd tools/probes/phase && python -c "import __graft_entry__ as g; g.build()")
"""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# (anchor, text inserted after the anchor) — each anchor must occur once
STAMPS = [
    ("  const int lane = threadIdx.x & 31;\n",
     "  unsigned long long* PH = p.tile_ts ? p.tile_ts + p.tiles + (size_t)blockIdx.x * 16 : nullptr;\n"
     "#define STAMP(i) do { if (PH) PH[i] = globaltimer(); } while (0)\n"
     "  if (threadIdx.x == 0) STAMP(0);\n"),
    ("    asm volatile(\"fence.mbarrier_init.release.cluster;\" ::: \"memory\");\n", "    STAMP(10);\n"),
    ("      asm volatile(\"tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\" ::: \"memory\");\n",
     "      if (lane == 0) STAMP(11);\n"),
    ("  const uint32_t tmem_base = *tmem_slot;\n", "  if (threadIdx.x == 0) STAMP(1);\n"),
    ("        stage = kk_pro % ST;\n", "        STAMP(2);\n"),
]


def patch(src):
    def once(a, b):
        nonlocal src
        assert src.count(a) == 1, (a, src.count(a))
        src = src.replace(a, b)
    once("  const int lane = threadIdx.x & 31;\n", STAMPS[0][0] + STAMPS[0][1])
    once(STAMPS[1][0], STAMPS[1][0] + STAMPS[1][1])
    once(STAMPS[2][0], STAMPS[2][0] + STAMPS[2][1])
    once(STAMPS[3][0], STAMPS[3][0] + STAMPS[3][1])
    once(STAMPS[4][0], STAMPS[4][1] + STAMPS[4][0])
    # MMA warp: first full barrier passed, last commit issued
    once("          mbar_wait(&full[stage], phase);\n          tc_fence_after();\n",
         "          mbar_wait(&full[stage], phase);\n          tc_fence_after();\n"
         "          if (k == 0 && kb == un.kb0 && lane == 0) STAMP(3);\n")
    once("        if (elect_one()) umma_commit<CG>(&tfull[acc], pair_mask);  // accumulator ready for the pair's epilogues\n"
         "        __syncwarp();\n",
         "        if (elect_one()) umma_commit<CG>(&tfull[acc], pair_mask);  // accumulator ready for the pair's epilogues\n"
         "        __syncwarp();\n        if (k == nu - 1 && lane == 0) STAMP(4);\n")
    # epilogue: last tile's accumulator ready, stores issued, signalled
    once("      const bool lte_tile = lte && k == nu - 1 && un.role == 0;\n",
         "      const bool lte_tile = lte && k == nu - 1 && un.role == 0;\n"
         "      if (k == nu - 1 && q == 0 && lane == 0) STAMP(5);\n")
    once("      if (p.tma_store && !owner && p.counters && lane == 0) {\n        bulk_wait_all();",
         "      if (k == nu - 1 && q == 0 && lane == 0) STAMP(6);\n"
         "      if (p.tma_store && !owner && p.counters && lane == 0) {\n        bulk_wait_all();")
    once("        if (p.tile_ts && leader) p.tile_ts[pos] = globaltimer();\n      }\n      if (++acc == 2) {",
         "        if (p.tile_ts && leader) p.tile_ts[pos] = globaltimer();\n        if (k == nu - 1) STAMP(7);\n"
         "      }\n      if (++acc == 2) {")
    once("  if (warp >= 4 && lane == 0 && p.tma_store) bulk_wait_all();  // the staging must outlive the stores\n",
         "  if (warp >= 4 && lane == 0 && p.tma_store) bulk_wait_all();  // the staging must outlive the stores\n"
         "  if (warp == 4 && lane == 0) STAMP(8);\n")
    once("  tc_fence_before();\n  if constexpr (CG * MC == 1) __syncthreads(); else cluster_sync();\n  if (warp == 2) {",
         "  tc_fence_before();\n  if constexpr (CG * MC == 1) __syncthreads(); else cluster_sync();\n"
         "  if (threadIdx.x == 0) STAMP(9);\n  if (warp == 2) {")
    # thread 0 reaches the setup barrier
    once("  tc_fence_before();\n  if constexpr (CG * MC == 1) __syncthreads(); else cluster_setup_sync();\n",
         "  if (threadIdx.x == 0) STAMP(12);\n"
         "  tc_fence_before();\n  if constexpr (CG * MC == 1) __syncthreads(); else cluster_setup_sync();\n")
    # prologue: first expect_tx, first stage's loads issued
    once("          if (leader) mbar_arrive_expect_tx(&full[s0], CG * C::STAGE_BYTES);\n",
         "          if (s0 == 0) STAMP(13);\n          if (leader) mbar_arrive_expect_tx(&full[s0], CG * C::STAGE_BYTES);\n")
    once("            tma_load_2d_2sm(sB + s0 * C::B_STAGE_BYTES, &tmB, s0 * BK, brow, fb);\n",
         "            tma_load_2d_2sm(sB + s0 * C::B_STAGE_BYTES, &tmB, s0 * BK, brow, fb);\n            if (s0 == 0) STAMP(14);\n")
    return src


def main():
    dest = sys.argv[1]
    if os.path.exists(dest):
        shutil.rmtree(dest)
    os.makedirs(dest)
    for d in ("paper_2504_19519_b200", "synthetic", "include"):
        shutil.copytree(os.path.join(ROOT, d), os.path.join(dest, d),
                        ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copy(os.path.join(ROOT, "__graft_entry__.py"), dest)
    f = os.path.join(dest, "paper_2504_19519_b200", "csrc", "kernels", "gemm_tcgen05.cu")
    src = open(f).read()
    open(f, "w").write(patch(src))


if __name__ == "__main__":
    main()
