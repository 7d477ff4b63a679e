// Host-side plan construction: see plan.h.  Every map here is checked
// element-by-element against oracle/ by tests/test_plan_parity.py.
#include "plan.h"

#include <algorithm>
#include <numeric>

namespace fo {

std::vector<int32_t> default_order(int Mt, int Nt, int s) {
  // DESIGN.md R1: row-panels of s tile-rows, panels top to
  // bottom, inside a panel column by column with the tile-row index fastest.
  std::vector<int32_t> o;
  o.reserve((size_t)Mt * Nt);
  for (int p0 = 0; p0 < Mt; p0 += s)
    for (int j = 0; j < Nt; ++j)
      for (int i = p0; i < std::min(p0 + s, Mt); ++i) o.push_back(i * Nt + j);
  return o;
}

// Generalized Hilbert curve over a w x h rectangle (any sizes; R44):
// consecutive positions are neighbouring tiles, so any run of S positions —
// a wave — covers a compact region and touches few tile-rows + tile-columns,
// whatever S is (a panel order's waves straddle panel boundaries unless S is a
// multiple of the panel size).  Recursive split of the longer side, as in
// J. Cervený's "gilbert" construction.
static int sgn(int v) { return (v > 0) - (v < 0); }
static int floordiv2(int v) { return v >= 0 ? v / 2 : -((-v + 1) / 2); }

static void gilbert(int x, int y, int ax, int ay, int bx, int by, int Nt, std::vector<int32_t>& out) {
  const int w = std::abs(ax + ay), h = std::abs(bx + by);
  const int dax = sgn(ax), day = sgn(ay), dbx = sgn(bx), dby = sgn(by);
  if (h == 1) {
    for (int i = 0; i < w; ++i, x += dax, y += day) out.push_back(y * Nt + x);
    return;
  }
  if (w == 1) {
    for (int i = 0; i < h; ++i, x += dbx, y += dby) out.push_back(y * Nt + x);
    return;
  }
  int ax2 = floordiv2(ax), ay2 = floordiv2(ay), bx2 = floordiv2(bx), by2 = floordiv2(by);
  const int w2 = std::abs(ax2 + ay2), h2 = std::abs(bx2 + by2);
  if (2 * w > 3 * h) {
    if ((w2 & 1) && w > 2) {
      ax2 += dax;
      ay2 += day;
    }
    gilbert(x, y, ax2, ay2, bx, by, Nt, out);
    gilbert(x + ax2, y + ay2, ax - ax2, ay - ay2, bx, by, Nt, out);
  } else {
    if ((h2 & 1) && h > 2) {
      bx2 += dbx;
      by2 += dby;
    }
    gilbert(x, y, bx2, by2, ax2, ay2, Nt, out);
    gilbert(x + bx2, y + by2, ax, ay, bx - bx2, by - by2, Nt, out);
    gilbert(x + (ax - dax) + (bx2 - dbx), y + (ay - day) + (by2 - dby), -bx2, -by2, -(ax - ax2), -(ay - ay2), Nt,
            out);
  }
}

std::vector<int32_t> hilbert_order(int Mt, int Nt) {
  std::vector<int32_t> o;
  o.reserve((size_t)Mt * Nt);
  if (Nt >= Mt) gilbert(0, 0, Nt, 0, 0, Mt, Nt, o);   // x = tile-column, y = tile-row
  else gilbert(0, 0, 0, Mt, Nt, 0, Nt, o);
  return o;
}

// Tile-rows + tile-columns touched, summed over the waves of S positions
// (stamp arrays: linear in the number of tiles).
static long order_footprint(const std::vector<int32_t>& o, int Nt, int S) {
  int Mt = 0;
  for (int32_t t : o) Mt = std::max(Mt, t / Nt + 1);
  std::vector<int32_t> rstamp((size_t)Mt, -1), cstamp((size_t)Nt, -1);
  long total = 0;
  for (size_t q = 0; q < o.size(); ++q) {
    const int32_t w = (int32_t)(q / (size_t)S);
    const int r = o[q] / Nt, c = o[q] % Nt;
    if (rstamp[(size_t)r] != w) {
      rstamp[(size_t)r] = w;
      ++total;
    }
    if (cstamp[(size_t)c] != w) {
      cstamp[(size_t)c] = w;
      ++total;
    }
  }
  return total;
}

// Footprint of the panel order of height s: tile-rows + tile-columns touched,
// summed over all waves (each touched row / column is an operand panel the
// wave streams from HBM; measured, the bench GEMM's DRAM reads follow it:
// 82 / 75 / 71 panels -> 526 / 490 / 468 MB, profiles/r02_order_probe.txt).
static long wave_footprint(int Mt, int Nt, int S, int s) {
  return order_footprint(default_order(Mt, Nt, s), Nt, S);
}

int auto_swizzle(int Mt, int Nt, int S) {
  int best = 1;
  long best_fp = -1;
  for (int s = 1; s <= Mt; ++s) {
    const long fp = wave_footprint(Mt, Nt, S, s);
    if (best_fp < 0 || fp < best_fp) {
      best_fp = fp;
      best = s;
    }
  }
  return best;
}

// AllReduce / ReduceScatter: prefer panel heights whose panels end exactly on
// the group boundaries (every group is then a band of whole tile-rows, panels
// top to bottom -> ROWBAND layout, no reorder at all) unless the
// unconstrained footprint is much smaller.
// The band-aligned panel height with the smallest wave footprint (-1: none).
static int band_swizzle(int Mt, int Nt, int S, const std::vector<int32_t>& gpos, long* fp_out) {
  int band = -1;
  long band_fp = -1;
  for (int s = 1; s <= Mt; ++s) {
    bool ok = true;
    for (size_t j = 1; j + 1 < gpos.size() && ok; ++j) ok = (gpos[j] % ((long)s * Nt) == 0);
    if (!ok) continue;
    const long fp = wave_footprint(Mt, Nt, S, s);
    if (band < 0 || fp < band_fp) {
      band = s;
      band_fp = fp;
    }
  }
  if (fp_out) *fp_out = band_fp;
  return band;
}

static int auto_swizzle_ar(int Mt, int Nt, int S, const std::vector<int32_t>& gpos) {
  const int any = auto_swizzle(Mt, Nt, S);
  long band_fp = -1;
  const int band = band_swizzle(Mt, Nt, S, gpos, &band_fp);
  if (band > 0 && 4 * band_fp <= 5 * wave_footprint(Mt, Nt, S, any)) return band;
  return any;
}

static void check_tile_shape(int BM, int BN) {
  if (BM != 64 && BM != 128 && BM != 256) fail(FO_ERR_UNSUPPORTED, "tile_m=%d not compiled (64, 128 or 256)", BM);
  if (BN != 64 && BN != 128 && BN != 256) fail(FO_ERR_UNSUPPORTED, "tile_n=%d not compiled (64/128/256)", BN);
}

struct Grid {
  int Mt, Nt, tiles, T, P;
  std::vector<int32_t> order, gpos, waves;
};

// O1-O3 for one descriptor (shared by self and A2A peers).
static Grid make_grid(const fo_plan_desc& d, int world) {
  // an All-to-All source with no rows (an expert rank no token was routed to)
  // still takes part in every group's exchange: m = 0, T = 0, P empty groups
  // (R45)
  const bool empty_src = d.coll == FO_ALLTOALL && d.m == 0;
  if ((d.m <= 0 && !empty_src) || d.n <= 0 || d.k <= 0) fail(FO_ERR_SHAPE, "m, n, k must be positive");
  check_tile_shape(d.tile_m, d.tile_n);
  if (d.m % d.tile_m || d.n % d.tile_n)
    fail(FO_ERR_SHAPE, "shape %lldx%lld not divisible by tile %dx%d", (long long)d.m, (long long)d.n,
         d.tile_m, d.tile_n);
  if (d.k % 64) fail(FO_ERR_SHAPE, "k=%lld must be a multiple of 64", (long long)d.k);
  if (d.workers < 1) fail(FO_ERR_INVALID_ARG, "workers (wave width S) must be >= 1");
  Grid g;
  g.Mt = (int)(d.m / d.tile_m);
  g.Nt = (int)(d.n / d.tile_n);
  g.tiles = g.Mt * g.Nt;
  // T = ceil(tiles / S) (Alg. 1 line 3)
  g.T = (g.tiles + d.workers - 1) / d.workers;
  if (d.group_waves && d.num_groups > 0) {
    g.waves.assign(d.group_waves, d.group_waves + d.num_groups);
  } else {
    g.waves.assign(1, g.T);
  }
  g.P = (int)g.waves.size();
  long sum = 0;
  for (int w : g.waves) {
    if (g.tiles > 0 && w < 1) fail(FO_ERR_INVALID_ARG, "group of %d waves (must be >= 1)", w);
    if (g.tiles == 0 && w != 0) fail(FO_ERR_INVALID_ARG, "a source with no rows has empty groups (0 waves each)");
    sum += w;
  }
  if (sum != g.T) fail(FO_ERR_INVALID_ARG, "group_waves sum to %ld but T=%d", sum, g.T);
  // group j = positions [S*W_{j-1}, min(S*W_j, tiles))
  g.gpos.assign(g.P + 1, 0);
  long W = 0;
  for (int j = 0; j < g.P; ++j) {
    W += g.waves[j];
    g.gpos[j + 1] = (int32_t)std::min<long>((long)d.workers * W, g.tiles);
  }
  if (g.tiles == 0) {
    g.order.clear();
  } else if (d.tile_order) {
    g.order.assign(d.tile_order, d.tile_order + g.tiles);
    std::vector<char> seen(g.tiles, 0);
    for (int32_t t : g.order) {
      if (t < 0 || t >= g.tiles || seen[t]) fail(FO_ERR_INVALID_ARG, "tile_order is not a permutation");
      seen[t] = 1;
    }
  } else if (d.swizzle == -1) {
    g.order = hilbert_order(g.Mt, g.Nt);  // DESIGN.md R44
  } else {
    if (d.swizzle < 0) fail(FO_ERR_INVALID_ARG, "swizzle must be >= -1");
    int s = d.swizzle;
    const bool autos = s == 0;
    if (s == 0) {
      // ROWBAND asked for: the best band-aligned panel height; AUTO (AR / RS):
      // band-aligned unless its footprint is much larger; otherwise (and
      // A2A AUTO) the footprint-minimal height
      const int band = d.ar_layout == FO_LAYOUT_ROWBAND ? band_swizzle(g.Mt, g.Nt, d.workers, g.gpos, nullptr) : -1;
      s = band > 0 ? band
          : ((d.coll == FO_ALLREDUCE || d.coll == FO_REDUCESCATTER) && d.ar_layout != FO_LAYOUT_SLOT)
              ? auto_swizzle_ar(g.Mt, g.Nt, d.workers, g.gpos)
              : auto_swizzle(g.Mt, g.Nt, d.workers);
    }
    g.order = default_order(g.Mt, g.Nt, s);
    if (autos) {
      // the generalized Hilbert order (R44) when it touches clearly fewer
      // operand panels over all waves and no band layout depends on the
      // panel order (one group is a band in any order; a panel height that is
      // not aligned to the groups gives no bands either)
      bool aligned = true;
      for (size_t j = 1; j + 1 < g.gpos.size() && aligned; ++j) aligned = g.gpos[j] % ((long)s * g.Nt) == 0;
      const bool band_pref = d.ar_layout != FO_LAYOUT_SLOT && d.coll != FO_NOCOMM;
      if (!band_pref || g.P == 1 || !aligned) {
        std::vector<int32_t> hil = hilbert_order(g.Mt, g.Nt);
        if (20 * order_footprint(hil, g.Nt, d.workers) < 19 * order_footprint(g.order, g.Nt, d.workers))
          g.order.swap(hil);
      }
    }
  }
  (void)world;
  return g;
}

// A2A send side of one source: pools per destination, subtokens
// appended in execution order (position p, then row a).  Returns, per
// destination d and group j, the (row, tile-col) list of that pool range.
struct A2ASide {
  std::vector<int64_t> cnt;    // [P*world]
  std::vector<int64_t> start;  // [P*world] start within pool d
  std::vector<int64_t> total;  // [world]
};

static A2ASide a2a_census(const fo_plan_desc& d, const Grid& g, int world) {
  A2ASide a;
  a.cnt.assign((size_t)g.P * world, 0);
  a.start.assign((size_t)g.P * world, 0);
  a.total.assign(world, 0);
  for (int j = 0; j < g.P; ++j) {
    for (int dd = 0; dd < world; ++dd) a.start[(size_t)j * world + dd] = a.total[dd];
    for (int p = g.gpos[j]; p < g.gpos[j + 1]; ++p) {
      int i = g.order[p] / g.Nt;
      for (int r = 0; r < d.tile_m; ++r) {
        int dst = d.row_dst[(int64_t)i * d.tile_m + r];
        a.cnt[(size_t)j * world + dst]++;
        a.total[dst]++;
      }
    }
  }
  return a;
}

// ROWBAND legality (H11a, R40): every group's tiles are exactly the
// complete tile-rows of one contiguous band [r0, r1) (any order inside); fills
// band_rows.  `ascending`: the bands must also follow each other top to bottom
// in group order (ReduceScatter: the receive buffer concatenates the groups'
// chunks, which is then the output itself).
static bool bands_of(int Mt, int Nt, int P, const std::vector<int32_t>& gpos, const std::vector<int32_t>& order,
                     bool ascending, std::vector<int64_t>* band_rows) {
  band_rows->assign(2 * P, 0);
  int64_t next = 0;
  for (int j = 0; j < P; ++j) {
    const int lo = gpos[j], hi = gpos[j + 1];
    if ((hi - lo) % Nt) return false;
    int rmin = Mt, rmax = -1;
    std::vector<char> seen((size_t)(hi - lo), 0);
    for (int q = lo; q < hi; ++q) rmin = std::min(rmin, order[q] / Nt);
    const int r1 = rmin + (hi - lo) / Nt;
    for (int q = lo; q < hi; ++q) {
      const int t = order[q] - rmin * Nt;
      if (t < 0 || t >= hi - lo || seen[t]) return false;
      seen[t] = 1;
      rmax = std::max(rmax, order[q] / Nt);
    }
    if (rmax >= r1) return false;
    if (ascending && rmin != next) return false;
    next = r1;
    (*band_rows)[2 * j] = rmin;
    (*band_rows)[2 * j + 1] = r1;
  }
  return true;
}

static bool band_layout(PlanHost& p, bool ascending) {
  return bands_of(p.Mt, p.Nt, p.P, p.gpos, p.order, ascending, &p.band_rows);
}

PlanHost build_plan(const fo_plan_desc& d, int rank, int world, const fo_plan_desc* const* peers,
                    int /*sm_count*/) {
  if (world < 1 || rank < 0 || rank >= world) fail(FO_ERR_INVALID_ARG, "rank %d / world %d", rank, world);
  if (d.coll < FO_ALLREDUCE || d.coll > FO_NOCOMM) fail(FO_ERR_INVALID_ARG, "unknown coll %d", d.coll);
  if (d.post < FO_POST_NONE || d.post > FO_POST_ADD_RMSNORM_RESIDUAL) fail(FO_ERR_INVALID_ARG, "unknown post %d", d.post);
  Grid g = make_grid(d, world);

  PlanHost p;
  p.coll = d.coll;
  p.M = d.m; p.N = d.n; p.K = d.k;
  p.BM = d.tile_m; p.BN = d.tile_n;
  p.S = d.workers;
  p.post = d.post;
  p.eps = d.eps;
  p.rank = rank; p.world = world;
  if (d.a_mn_major < 0 || d.a_mn_major > 1 || d.b_mn_major < 0 || d.b_mn_major > 1)
    fail(FO_ERR_INVALID_ARG, "a_mn_major / b_mn_major must be 0 or 1");
  p.mn_major = (d.a_mn_major ? 1 : 0) | (d.b_mn_major ? 2 : 0);
  if (p.mn_major && p.BN < 128) fail(FO_ERR_UNSUPPORTED, "MN-major operands need tile_n >= 128");
  p.Mt = g.Mt; p.Nt = g.Nt; p.tiles = g.tiles; p.T = g.T; p.P = g.P;
  p.order = g.order;
  p.group_waves = g.waves;
  p.gpos = g.gpos;
  p.pos_of_tile.assign(p.tiles, 0);
  for (int q = 0; q < p.tiles; ++q) p.pos_of_tile[p.order[q]] = q;
  p.group_of_pos.assign(p.tiles, 0);
  for (int j = 0; j < p.P; ++j)
    for (int q = p.gpos[j]; q < p.gpos[j + 1]; ++q) p.group_of_pos[q] = j;

  const int64_t MN = p.M * p.N;
  switch (p.coll) {
    case FO_NOCOMM:
      p.layout = FO_LAYOUT_ROWBAND;
      p.out_rows = p.M;
      p.send_elems = p.recv_elems = MN;
      break;
    case FO_ALLREDUCE: {
      // ROWBAND (H11a) is legal iff every group's tiles are exactly
      // the complete tile-rows of one contiguous band [r0, r1) (any order inside).
      const bool ok = band_layout(p, false);
      if (d.ar_layout == FO_LAYOUT_ROWBAND && !ok)
        fail(FO_ERR_UNSUPPORTED, "ROWBAND layout needs a raster order and tile-row group boundaries");
      p.layout = (d.ar_layout == FO_LAYOUT_SLOT) ? FO_LAYOUT_SLOT
                 : ok                           ? FO_LAYOUT_ROWBAND
                                                : FO_LAYOUT_SLOT;
      p.out_rows = p.M;
      p.send_elems = p.recv_elems = MN;
      break;
    }
    case FO_REDUCESCATTER: {
      // subtile of h = BM/n rows (R7)
      if (p.BM % world) fail(FO_ERR_SHAPE, "tile_m=%d not divisible by world=%d", p.BM, world);
      p.h = p.BM / world;
      p.out_rows = p.M / world;
      p.send_elems = MN;
      // ROWBAND (R40): ascending bands of whole tile-rows; chunk k
      // of a band = the k-th subtile rows of its tiles as complete rows, so
      // the ReduceScatter delivers the output rows in place (no receive buffer)
      const bool ok = d.ar_layout != FO_LAYOUT_SLOT && band_layout(p, true);
      if (d.ar_layout == FO_LAYOUT_ROWBAND && !ok)
        fail(FO_ERR_UNSUPPORTED, "RS ROWBAND layout needs ascending bands of whole tile-rows as groups");
      p.layout = ok ? FO_LAYOUT_ROWBAND : FO_LAYOUT_SLOT;
      if (!ok) p.band_rows.clear();
      p.recv_elems = MN / world;
      break;
    }
    case FO_ALLTOALL: {
      if (!d.row_dst && p.M > 0) fail(FO_ERR_INVALID_ARG, "All-to-All needs row_dst");
      for (int64_t r = 0; r < p.M; ++r)
        if (d.row_dst[r] < 0 || d.row_dst[r] >= world) fail(FO_ERR_INVALID_ARG, "row_dst[%lld] out of range", (long long)r);
      if (p.M > 0) p.row_dst.assign(d.row_dst, d.row_dst + p.M);
      // ---- every source's grid (the census exchange: peers' descriptors)
      if (!peers) fail(FO_ERR_INVALID_ARG, "All-to-All needs the peers' descriptors");
      std::vector<Grid> pg(world);
      for (int s = 0; s < world; ++s) {
        const fo_plan_desc* ps = (s == rank) ? &d : peers[s];
        if (!ps) fail(FO_ERR_INVALID_ARG, "peer %d descriptor missing", s);
        if (ps->n != d.n || ps->tile_n != d.tile_n || ps->tile_m != d.tile_m)
          fail(FO_ERR_INVALID_ARG, "peer %d: n / tile shape differ", s);
        if (!ps->row_dst && ps->m > 0) fail(FO_ERR_INVALID_ARG, "peer %d: row_dst missing", s);
        pg[s] = make_grid(*ps, world);
        if (pg[s].P != p.P) fail(FO_ERR_INVALID_ARG, "peer %d has %d groups, self %d", s, pg[s].P, p.P);
      }
      // ROWBAND (R41): every source asks for it (or AUTO) and every
      // source's groups are ascending bands of whole tile-rows — decided from
      // the same descriptors on every rank, so senders and receivers agree
      bool band = true;
      std::vector<std::vector<int64_t>> bands(world);
      for (int s = 0; s < world && band; ++s) {
        const fo_plan_desc* ps = (s == rank) ? &d : peers[s];
        band = ps->ar_layout != FO_LAYOUT_SLOT &&
               bands_of(pg[s].Mt, pg[s].Nt, pg[s].P, pg[s].gpos, pg[s].order, true, &bands[s]);
      }
      if (d.ar_layout == FO_LAYOUT_ROWBAND && !band)
        fail(FO_ERR_UNSUPPORTED, "A2A ROWBAND layout needs every source's groups to be ascending bands of whole tile-rows");
      p.layout = band ? FO_LAYOUT_ROWBAND : FO_LAYOUT_SLOT;
      if (band) p.band_rows = bands[rank];
      // ---- send side (self)
      A2ASide me = a2a_census(d, g, world);
      p.send_cnt = me.cnt;
      p.send_start = me.start;
      p.pool_base.assign(world + 1, 0);
      for (int dd = 0; dd < world; ++dd) p.pool_base[dd + 1] = p.pool_base[dd] + me.total[dd];
      p.send_elems = p.pool_base[world] * p.BN;
      p.row_slot.assign((size_t)p.tiles * p.BM, -1);
      {
        std::vector<int64_t> fill(world, 0);
        if (band) {
          // pool d: complete rows, source row ascending (bands ascending), then
          // tile-column: subtoken (row, jc) of tile (row/BM, jc) at position q
          for (int64_t r = 0; r < p.M; ++r) {
            const int dst = p.row_dst[r];
            const int i = (int)(r / p.BM);
            for (int jc = 0; jc < p.Nt; ++jc) {
              const int q = p.pos_of_tile[i * p.Nt + jc];
              p.row_slot[(size_t)q * p.BM + r % p.BM] = (int32_t)(p.pool_base[dst] + fill[dst]++);
            }
          }
        } else {
          for (int q = 0; q < p.tiles; ++q) {
            int i = p.order[q] / p.Nt;
            for (int r = 0; r < p.BM; ++r) {
              int dst = p.row_dst[(int64_t)i * p.BM + r];
              p.row_slot[(size_t)q * p.BM + r] = (int32_t)(p.pool_base[dst] + fill[dst]++);
            }
          }
        }
      }
      // output rows: sources ascending, then source rows ascending (all-to-all-v order)
      p.src_base.assign(world + 1, 0);
      std::vector<std::vector<int32_t>> rank_of_row(world);
      for (int s = 0; s < world; ++s) {
        const fo_plan_desc* ps = (s == rank) ? &d : peers[s];
        rank_of_row[s].assign(ps->m, -1);
        int64_t c = 0;
        for (int64_t r = 0; r < ps->m; ++r)
          if (ps->row_dst[r] == rank) rank_of_row[s][r] = (int32_t)c++;
        p.src_base[s + 1] = p.src_base[s] + c;
      }
      p.out_rows = p.src_base[world];
      // receive layout [group j][source s] (R9); ROWBAND: the output
      // itself — group j's rows from source s are the run of output rows
      // starting at the first of them (R41)
      p.recv_cnt.assign((size_t)p.P * world, 0);
      p.recv_off.assign((size_t)p.P * world, 0);
      std::vector<A2ASide> sides(world);
      for (int s = 0; s < world; ++s) {
        const fo_plan_desc* ps = (s == rank) ? &d : peers[s];
        sides[s] = a2a_census(*ps, pg[s], world);
      }
      if (band) {
        for (int j = 0; j < p.P; ++j)
          for (int s = 0; s < world; ++s) {
            const fo_plan_desc* ps = (s == rank) ? &d : peers[s];
            p.recv_cnt[(size_t)j * world + s] = sides[s].cnt[(size_t)j * world + rank];
            const int64_t b0 = bands[s][2 * j] * ps->tile_m, b1 = bands[s][2 * j + 1] * ps->tile_m;
            int64_t first = -1;
            for (int64_t r = b0; r < b1 && first < 0; ++r)
              if (ps->row_dst[r] == rank) first = rank_of_row[s][r];
            p.recv_off[(size_t)j * world + s] = first < 0 ? 0 : (p.src_base[s] + first) * p.Nt;
          }
        p.recv_elems = p.out_rows * p.N;
        p.src_row.resize((size_t)p.out_rows * p.Nt);
        p.recv_dst.resize((size_t)p.out_rows * p.Nt);
        for (int64_t x = 0; x < p.out_rows * p.Nt; ++x) p.src_row[(size_t)x] = p.recv_dst[(size_t)x] = (int32_t)x;
        break;
      }
      int64_t off = 0;
      for (int j = 0; j < p.P; ++j)
        for (int s = 0; s < world; ++s) {
          p.recv_off[(size_t)j * world + s] = off;
          p.recv_cnt[(size_t)j * world + s] = sides[s].cnt[(size_t)j * world + rank];
          off += sides[s].cnt[(size_t)j * world + rank];
        }
      p.recv_elems = off * p.BN;
      p.src_row.assign((size_t)p.out_rows * p.Nt, -1);
      p.recv_dst.assign((size_t)off, -1);
      for (int s = 0; s < world; ++s) {
        const fo_plan_desc* ps = (s == rank) ? &d : peers[s];
        const Grid& gs = pg[s];
        for (int j = 0; j < gs.P; ++j) {
          int64_t idx = p.recv_off[(size_t)j * world + s];
          for (int q = gs.gpos[j]; q < gs.gpos[j + 1]; ++q) {
            int i = gs.order[q] / gs.Nt, jc = gs.order[q] % gs.Nt;
            for (int r = 0; r < ps->tile_m; ++r) {
              int64_t row = (int64_t)i * ps->tile_m + r;
              if (ps->row_dst[row] != rank) continue;
              int64_t orow = p.src_base[s] + rank_of_row[s][row];
              p.recv_dst[(size_t)idx] = (int32_t)(orow * p.Nt + jc);
              p.src_row[(size_t)orow * p.Nt + jc] = (int32_t)idx++;
            }
          }
        }
      }
      break;
    }
  }
  if (p.coll == FO_NOCOMM) p.layout = FO_LAYOUT_ROWBAND;
  build_schedules(p, d, peers);
  return p;
}

static fo_comm_call make_call(int kind, int group, int peer, int sbuf, int dbuf, int64_t soff, int64_t doff,
                              int64_t count) {
  fo_comm_call c{};
  c.kind = kind;
  c.group = group;
  c.peer = peer;
  c.src_buf = sbuf;
  c.dst_buf = dbuf;
  c.src_off = soff;
  c.dst_off = doff;
  c.count = count;
  return c;
}

// Maximal runs [r0, r1) of consecutive rows of `row_dst[0..m)` with destination `dst`.
static std::vector<std::pair<int64_t, int64_t>> dst_runs(const int32_t* row_dst, int64_t m, int dst) {
  std::vector<std::pair<int64_t, int64_t>> runs;
  for (int64_t r = 0; r < m;) {
    if (row_dst[r] != dst) {
      ++r;
      continue;
    }
    int64_t e = r;
    while (e < m && row_dst[e] == dst) ++e;
    runs.emplace_back(r, e);
    r = e;
  }
  return runs;
}

void build_schedules(PlanHost& p, const fo_plan_desc& d, const fo_plan_desc* const* peers) {
  p.calls.clear();
  p.seq_calls.clear();
  p.call_begin.assign(p.P + 1, 0);
  const int W = p.world;
  // ---- overlapped (fo_run): one call set per wave group, on the group's
  // contiguous range
  for (int j = 0; j < p.P; ++j) {
    p.call_begin[j] = (int32_t)p.calls.size();
    switch (p.coll) {
      case FO_ALLREDUCE: {
        // in place: ROWBAND reduces the group's row band of the caller's C,
        // SLOT the group's slots of the send buffer
        const int buf = (p.layout == FO_LAYOUT_ROWBAND) ? FO_BUF_OUT : FO_BUF_SEND;
        const int64_t b = p.group_elem_begin(j), e = p.group_elem_end(j);
        p.calls.push_back(make_call(FO_CALL_ALLREDUCE, j, -1, buf, buf, b, b, e - b));
        break;
      }
      case FO_REDUCESCATTER: {
        // chunk k of the group's range goes to rank k; rank k's chunks are
        // stored in group order (receive layout [group][q][a'][BN]); ROWBAND:
        // straight into the output rows of the band (at one rank the GEMM
        // writes the output itself and the call is in place)
        const int64_t b = p.group_elem_begin(j), e = p.group_elem_end(j);
        const bool band = p.layout == FO_LAYOUT_ROWBAND;
        p.calls.push_back(make_call(FO_CALL_REDUCESCATTER, j, -1, band && W == 1 ? FO_BUF_OUT : FO_BUF_SEND,
                                    band ? FO_BUF_OUT : FO_BUF_RECV, b, b / W, (e - b) / W));
        break;
      }
      case FO_ALLTOALL: {
        // the self part is a local copy; every peer's part of pool d in one
        // grouped send/recv
        const int64_t cs = p.send_cnt[(size_t)j * W + p.rank];
        if (cs)
          p.calls.push_back(make_call(FO_CALL_LOCAL_COPY, j, p.rank, FO_BUF_SEND, FO_BUF_RECV,
                                      (p.pool_base[p.rank] + p.send_start[(size_t)j * W + p.rank]) * p.BN,
                                      p.recv_off[(size_t)j * W + p.rank] * p.BN, cs * p.BN));
        p.calls.push_back(make_call(FO_CALL_GROUP_START, j, -1, FO_BUF_NONE, FO_BUF_NONE, 0, 0, 0));
        for (int dd = 0; dd < W; ++dd) {
          if (dd == p.rank) continue;
          const int64_t sc = p.send_cnt[(size_t)j * W + dd];
          if (sc)
            p.calls.push_back(make_call(FO_CALL_SEND, j, dd, FO_BUF_SEND, FO_BUF_NONE,
                                        (p.pool_base[dd] + p.send_start[(size_t)j * W + dd]) * p.BN, 0, sc * p.BN));
          const int64_t rc = p.recv_cnt[(size_t)j * W + dd];
          if (rc)
            p.calls.push_back(make_call(FO_CALL_RECV, j, dd, FO_BUF_NONE, FO_BUF_RECV, 0,
                                        p.recv_off[(size_t)j * W + dd] * p.BN, rc * p.BN));
        }
        p.calls.push_back(make_call(FO_CALL_GROUP_END, j, -1, FO_BUF_NONE, FO_BUF_NONE, 0, 0, 0));
        break;
      }
      default:
        break;
    }
  }
  p.call_begin[p.P] = (int32_t)p.calls.size();
  // ---- sequential baseline (fo_run_sequential): one full-size call
  const int64_t MN = p.M * p.N;
  switch (p.coll) {
    case FO_ALLREDUCE:
      p.seq_calls.push_back(make_call(FO_CALL_ALLREDUCE, -1, -1, FO_BUF_OUT, FO_BUF_OUT, 0, 0, MN));
      break;
    case FO_REDUCESCATTER:
      p.seq_calls.push_back(make_call(FO_CALL_REDUCESCATTER, -1, -1, FO_BUF_SCRATCH, FO_BUF_OUT, 0, 0, MN / W));
      break;
    case FO_ALLTOALL: {
      // rows of row-major C in runs of one destination; a source's rows land
      // at out rows src_base[s] + (their rank among its rows routed here)
      auto desc = [&](int s) { return s == p.rank ? &d : peers[s]; };
      std::vector<std::vector<fo_comm_call>> sends(W), recvs(W);
      for (int dd = 0; dd < W; ++dd)
        for (auto& rr : dst_runs(d.row_dst, d.m, dd))
          sends[dd].push_back(make_call(FO_CALL_SEND, -1, dd, FO_BUF_SCRATCH, FO_BUF_NONE, rr.first * p.N, 0,
                                        (rr.second - rr.first) * p.N));
      for (int s = 0; s < W; ++s) {
        int64_t o = p.src_base[s];
        for (auto& rr : dst_runs(desc(s)->row_dst, desc(s)->m, p.rank)) {
          recvs[s].push_back(make_call(FO_CALL_RECV, -1, s, FO_BUF_NONE, FO_BUF_OUT, 0, o * p.N,
                                       (rr.second - rr.first) * p.N));
          o += rr.second - rr.first;
        }
      }
      // self part: local copies run by run
      for (size_t i = 0; i < sends[p.rank].size(); ++i) {
        fo_comm_call c = sends[p.rank][i];
        c.kind = FO_CALL_LOCAL_COPY;
        c.dst_buf = FO_BUF_OUT;
        c.dst_off = recvs[p.rank][i].dst_off;
        p.seq_calls.push_back(c);
      }
      p.seq_calls.push_back(make_call(FO_CALL_GROUP_START, -1, -1, FO_BUF_NONE, FO_BUF_NONE, 0, 0, 0));
      for (int dd = 0; dd < W; ++dd) {
        if (dd == p.rank) continue;
        for (auto& c : sends[dd]) p.seq_calls.push_back(c);
        for (auto& c : recvs[dd]) p.seq_calls.push_back(c);
      }
      p.seq_calls.push_back(make_call(FO_CALL_GROUP_END, -1, -1, FO_BUF_NONE, FO_BUF_NONE, 0, 0, 0));
      break;
    }
    default:
      break;
  }
}

int64_t PlanHost::send_index(int64_t r, int64_t c) const {
  const int i = (int)(r / BM), a = (int)(r % BM), jc = (int)(c / BN), b = (int)(c % BN);
  const int q = pos_of_tile[i * Nt + jc];
  switch (coll) {
    case FO_NOCOMM:
      return r * N + c;
    case FO_ALLREDUCE:
      if (layout == FO_LAYOUT_ROWBAND) return r * N + c;
      return ((int64_t)q * BM + a) * BN + b;  // slot q, row-major
    case FO_REDUCESCATTER: {
      const int j = group_of_pos[q];
      const int k = a / h, a2 = a % h;
      if (layout == FO_LAYOUT_ROWBAND) {  // DESIGN.md R40
        const int64_t r0 = band_rows[2 * j], B = band_rows[2 * j + 1] - r0;
        return (r0 * BM + (k * B + (i - r0)) * h + a2) * N + c;
      }
      const int ps = gpos[j], G = gpos[j + 1] - gpos[j];
      return (int64_t)ps * BM * BN + (int64_t)k * G * h * BN + (int64_t)(q - ps) * h * BN + (int64_t)a2 * BN + b;
    }
    case FO_ALLTOALL:
      return (int64_t)row_slot[(size_t)q * BM + a] * BN + b;
  }
  return -1;
}

int64_t PlanHost::recv_index(int64_t r, int64_t c) const {
  const int jc = (int)(c / BN), b = (int)(c % BN);
  switch (coll) {
    case FO_NOCOMM:
      return r * N + c;
    case FO_ALLREDUCE: {
      if (layout == FO_LAYOUT_ROWBAND) return r * N + c;
      const int q = pos_of_tile[(r / BM) * Nt + jc];
      return ((int64_t)q * BM + r % BM) * BN + b;
    }
    case FO_REDUCESCATTER: {
      if (layout == FO_LAYOUT_ROWBAND) return r * N + c;  // received in output order (R40)
      // local row l = i*h + a'  <-  receive row q*h + a' (group chunks in order)
      const int q = pos_of_tile[(r / h) * Nt + jc];
      return ((int64_t)q * h + r % h) * BN + b;
    }
    case FO_ALLTOALL:
      return (int64_t)src_row[(size_t)r * Nt + jc] * BN + b;
  }
  return -1;
}

}  // namespace fo
