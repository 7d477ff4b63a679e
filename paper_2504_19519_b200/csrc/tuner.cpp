// Alg. 1 "Grouping tuning algorithm": latency predictor
// and pruned predictive search over wave-group partitions.  Host only.
//
// Readings: R13 the first group's predecessor has 0 comm latency;
// R14 duration is measured at the actual wave width S, T = ceil(tiles/S);
// R15 bandwidth is linear in log2(bytes) between samples, clamped; R16 ties go
// to fewer groups, then the lexicographically smaller partition.
#include <cmath>
#include <functional>
#include <memory>
#include <limits>
#include <vector>

#include "common.h"

namespace fo {

struct Curve {
  std::vector<double> lx, bw;
  double latency_us(double bytes) const {
    if (bytes <= 0) return 0.0;
    const double x = std::log2(bytes);
    double b;
    if (x <= lx.front()) b = bw.front();
    else if (x >= lx.back()) b = bw.back();
    else {
      size_t k = 0;
      while (!(lx[k] <= x && x <= lx[k + 1])) ++k;
      const double f = (x - lx[k]) / (lx[k + 1] - lx[k]);
      b = bw[k] + f * (bw[k + 1] - bw[k]);
    }
    return bytes / (b * 1e9) * 1e6;
  }
};

static Curve make_curve(const double* bytes, const double* gbps, int n) {
  if (n < 1 || !bytes || !gbps) fail(FO_ERR_INVALID_ARG, "empty bandwidth curve");
  Curve c;
  for (int i = 0; i < n; ++i) {
    if (bytes[i] <= 0 || gbps[i] <= 0) fail(FO_ERR_INVALID_ARG, "curve point %d not positive", i);
    if (i && bytes[i] <= bytes[i - 1]) fail(FO_ERR_INVALID_ARG, "curve sizes must increase");
    c.lx.push_back(std::log2(bytes[i]));
    c.bw.push_back(gbps[i]);
  }
  return c;
}

// Lines 10-22 of Alg. 1 for one candidate.
static double predict(const std::vector<int>& G, double duration, int T, int tiles, int S, double tile_bytes,
                      const Curve& c) {
  auto size_of = [&](int i) {  // get_data_size(G_i): tiles of group i x bytes per tile
    long W0 = 0;
    for (int q = 0; q < i; ++q) W0 += G[q];
    const long lo = (long)S * W0, hi = std::min<long>((long)S * (W0 + G[i]), tiles);
    return (double)(hi - lo) * tile_bytes;
  };
  double acc_p = 0.0, acc_m = 0.0;
  for (size_t i = 0; i < G.size(); ++i) {
    const double t_m = i ? c.latency_us(size_of((int)i - 1)) : 0.0;
    const double t_p = duration / T * G[i];
    acc_m = std::max(acc_p, acc_m) + t_m;
    acc_p = acc_p + t_p;
  }
  return std::max(acc_p, acc_m) + c.latency_us(size_of((int)G.size() - 1));
}

// Exact argmin of the Alg. 1 predictor by dynamic programming (our
// extension for large T, where 2^(T-1) candidates cannot be enumerated).
// With E(w) the predicted end of the communication of the group that ends at
// wave w, lines 12-18 of Alg. 1 unroll to
//   E(w) = max(dur*w'/T, E(w')) + lat(bytes(w', w)),   E(0) = 0  (R13)
// where w' is the end of the previous group (the max takes the compute end of
// the group and the end of the previous communication), and lines 20-21 give
// the prediction E(T).  E is nondecreasing in E(w'), so the minimum over
// partitions is  E*(w) = min_{w'} max(dur*w'/T, E*(w')) + lat(w', w).
// Caps: first group <= s1 waves, last group <= sp waves (pruning).
static std::vector<int> dp_search(double duration, int T, int tiles, int S, double tile_bytes, const Curve& c,
                                  int s1, int sp, bool prune, double* best_t) {
  const double inf = std::numeric_limits<double>::infinity();
  auto bytes = [&](int w0, int w1) {
    const long lo = (long)S * w0, hi = std::min<long>((long)S * w1, tiles);
    return (double)(hi - lo) * tile_bytes;
  };
  std::vector<double> E(T + 1, inf);
  std::vector<int> prev(T + 1, -1), ng(T + 1, 0);
  E[0] = 0.0;
  for (int w = 1; w <= T; ++w) {
    for (int w0 = 0; w0 < w; ++w0) {
      if (E[w0] == inf) continue;
      if (prune && w0 == 0 && w > s1 && T > 1) continue;
      if (prune && w == T && (w - w0) > sp && T > 1) continue;
      const double start = (w0 == 0) ? 0.0 : std::max(duration * w0 / T, E[w0]);
      // the group's own comm is charged when the next group starts (or at the
      // end); E(w) below is the end of this group's communication
      const double e = std::max(duration * w / T, start) + c.latency_us(bytes(w0, w));
      if (e < E[w] || (e == E[w] && ng[w0] + 1 < ng[w])) {
        E[w] = e;
        prev[w] = w0;
        ng[w] = ng[w0] + 1;
      }
    }
  }
  if (!(E[T] < inf)) fail(FO_ERR_INVALID_ARG, "pruning left no candidate (s1=%d, sp=%d, T=%d)", s1, sp, T);
  std::vector<int> G;
  for (int w = T; w > 0; w = prev[w]) G.insert(G.begin(), w - prev[w]);
  *best_t = E[T];
  return G;
}

// ---- generic form: group latency lat(w0, w1) of the group covering waves [w0, w1)
using GroupLat = std::function<double(int, int)>;

static double predict_g(const std::vector<int>& G, double duration, int T, const GroupLat& lat) {
  double acc_p = 0.0, acc_m = 0.0;
  int W = 0, Wprev = 0;
  for (size_t i = 0; i < G.size(); ++i) {
    const double t_m = i ? lat(Wprev, W) : 0.0;
    acc_m = std::max(acc_p, acc_m) + t_m;
    acc_p += duration / T * G[i];
    Wprev = W;
    W += G[i];
  }
  return std::max(acc_p, acc_m) + lat(Wprev, W);
}

static std::vector<int> dp_g(double duration, int T, const GroupLat& lat, int s1, int sp, bool caps, double* best) {
  const double inf = std::numeric_limits<double>::infinity();
  std::vector<double> E(T + 1, inf);
  std::vector<int> prev(T + 1, -1), ng(T + 1, 0);
  E[0] = 0.0;
  for (int w = 1; w <= T; ++w)
    for (int w0 = 0; w0 < w; ++w0) {
      if (E[w0] == inf) continue;
      if (caps && T > 1 && ((w0 == 0 && w > s1) || (w == T && w - w0 > sp))) continue;
      const double e = std::max(duration * w / T, E[w0]) + lat(w0, w);
      if (e < E[w] || (e == E[w] && ng[w0] + 1 < ng[w])) {
        E[w] = e;
        prev[w] = w0;
        ng[w] = ng[w0] + 1;
      }
    }
  if (!(E[T] < inf)) fail(FO_ERR_INVALID_ARG, "pruning left no candidate (s1=%d, sp=%d, T=%d)", s1, sp, T);
  std::vector<int> G;
  for (int w = T; w > 0; w = prev[w]) G.insert(G.begin(), w - prev[w]);
  *best = E[T];
  return G;
}

static std::vector<int> enum_g(double duration, int T, const GroupLat& lat, int s1, int sp, bool prune, double* best_t) {
  std::vector<int> best, G;
  *best_t = std::numeric_limits<double>::infinity();
  for (uint32_t mask = 0; mask < (1u << (T - 1)); ++mask) {
    G.clear();
    int run = 0;
    for (int w = 0; w < T; ++w) {
      ++run;
      if (w == T - 1 || ((mask >> w) & 1u)) {
        G.push_back(run);
        run = 0;
      }
    }
    if (prune && T > 1 && (G.front() > s1 || G.back() > sp)) continue;
    const double t = predict_g(G, duration, T, lat);
    if (best.empty() || t < *best_t || (t == *best_t && (G.size() < best.size() || (G.size() == best.size() && G < best)))) {
      best = G;
      *best_t = t;
    }
  }
  return best;
}

// A2A imbalance extension (R26): all ranks share the
// wave partition; the accumulated compute is the maximum over ranks (=
// max duration) and a group's communication lasts as long as the slowest
// rank's message: lat(w0, w1) = max_r latency(sum of rank r's bytes of waves [w0, w1)).
static GroupLat multi_lat(int ranks, int T, const double* wave_bytes, const Curve* c) {
  auto prefix = std::make_shared<std::vector<double>>((size_t)ranks * (T + 1), 0.0);
  for (int r = 0; r < ranks; ++r)
    for (int w = 0; w < T; ++w)
      (*prefix)[(size_t)r * (T + 1) + w + 1] = (*prefix)[(size_t)r * (T + 1) + w] + wave_bytes[(size_t)r * T + w];
  return [prefix, ranks, T, c](int w0, int w1) {
    double m = 0.0;
    for (int r = 0; r < ranks; ++r) {
      const double b = (*prefix)[(size_t)r * (T + 1) + w1] - (*prefix)[(size_t)r * (T + 1) + w0];
      m = std::max(m, c->latency_us(b));
    }
    return m;
  };
}

}  // namespace fo

using namespace fo;

extern "C" fo_status fo_tune_predict_multi(const int32_t* groups, int32_t P, int32_t ranks, int32_t T,
                                           const double* durations, const double* wave_bytes,
                                           const double* curve_bytes, const double* curve_gbps, int32_t npts,
                                           double* predicted_us) {
  return guard([&] {
    if (!groups || P < 1 || ranks < 1 || T < 1 || !durations || !wave_bytes || !predicted_us)
      fail(FO_ERR_INVALID_ARG, "bad arguments");
    std::vector<int> G(groups, groups + P);
    long sum = 0;
    for (int g : G) {
      if (g < 1) fail(FO_ERR_INVALID_ARG, "zero-size group");
      sum += g;
    }
    if (sum != T) fail(FO_ERR_INVALID_ARG, "groups sum to %ld, T=%d", sum, T);
    const Curve c = make_curve(curve_bytes, curve_gbps, npts);
    double dmax = 0.0;
    for (int r = 0; r < ranks; ++r) dmax = std::max(dmax, durations[r]);
    *predicted_us = predict_g(G, dmax, T, multi_lat(ranks, T, wave_bytes, &c));
  });
}

extern "C" fo_status fo_tune_search_multi(int32_t ranks, int32_t T, const double* durations, const double* wave_bytes,
                                          const double* curve_bytes, const double* curve_gbps, int32_t npts,
                                          int32_t s1, int32_t sp, int32_t prune, int32_t* out_groups,
                                          int32_t* out_num_groups, double* predicted_us) {
  return guard([&] {
    if (ranks < 1 || T < 1 || !durations || !wave_bytes || !out_groups || !out_num_groups || !predicted_us)
      fail(FO_ERR_INVALID_ARG, "bad arguments");
    if (prune != 0 && (s1 < 1 || sp < 1)) fail(FO_ERR_INVALID_ARG, "pruning caps s1=%d, sp=%d must be >= 1", s1, sp);
    const Curve c = make_curve(curve_bytes, curve_gbps, npts);
    double dmax = 0.0;
    for (int r = 0; r < ranks; ++r) dmax = std::max(dmax, durations[r]);
    const GroupLat lat = multi_lat(ranks, T, wave_bytes, &c);
    double t = 0.0;
    std::vector<int> G = (prune >= 2 || T > 20)
                             ? dp_g(dmax, T, lat, s1, sp, prune == 1 || prune == 3, &t)
                             : enum_g(dmax, T, lat, s1, sp, prune != 0, &t);
    if (G.empty()) fail(FO_ERR_INVALID_ARG, "pruning left no candidate");
    for (size_t i = 0; i < G.size(); ++i) out_groups[i] = G[i];
    *out_num_groups = (int32_t)G.size();
    *predicted_us = predict_g(G, dmax, T, lat);
  });
}

extern "C" fo_status fo_tune_predict(const int32_t* groups, int32_t P, double duration_us, int32_t tiles,
                                     int32_t S, double tile_bytes, const double* curve_bytes,
                                     const double* curve_gbps, int32_t npts, double* predicted_us) {
  return guard([&] {
    if (!groups || P < 1 || !predicted_us || S < 1 || tiles < 1) fail(FO_ERR_INVALID_ARG, "bad arguments");
    const int T = (tiles + S - 1) / S;
    std::vector<int> G(groups, groups + P);
    long sum = 0;
    for (int g : G) {
      if (g < 1) fail(FO_ERR_INVALID_ARG, "zero-size group");
      sum += g;
    }
    if (sum != T) fail(FO_ERR_INVALID_ARG, "groups sum to %ld, T=%d", sum, T);
    *predicted_us = predict(G, duration_us, T, tiles, S, tile_bytes, make_curve(curve_bytes, curve_gbps, npts));
  });
}

extern "C" fo_status fo_tune_search(double duration_us, int32_t tiles, int32_t S, double tile_bytes,
                                    const double* curve_bytes, const double* curve_gbps, int32_t npts,
                                    int32_t s1, int32_t sp, int32_t prune, int32_t* out_groups,
                                    int32_t* out_num_groups, double* predicted_us) {
  return guard([&] {
    if (!out_groups || !out_num_groups || !predicted_us || S < 1 || tiles < 1) fail(FO_ERR_INVALID_ARG, "bad arguments");
    if (prune != 0 && (s1 < 1 || sp < 1)) fail(FO_ERR_INVALID_ARG, "pruning caps s1=%d, sp=%d must be >= 1", s1, sp);
    const int T = (tiles + S - 1) / S;
    const Curve c = make_curve(curve_bytes, curve_gbps, npts);
    if (prune >= 2 || T > 20) {
      // exact DP argmin (prune 2: all partitions, 3: with the caps; T > 20: caps iff prune == 1)
      const bool caps = (prune == 3) || (prune == 1);
      double t = 0;
      std::vector<int> G = dp_search(duration_us, T, tiles, S, tile_bytes, c, s1, sp, caps, &t);
      for (size_t i = 0; i < G.size(); ++i) out_groups[i] = G[i];
      *out_num_groups = (int32_t)G.size();
      *predicted_us = predict(G, duration_us, T, tiles, S, tile_bytes, c);
      return;
    }
    std::vector<int> best;
    double best_t = std::numeric_limits<double>::infinity();
    std::vector<int> G;
    // line 7: the binary communicate/not decision after each wave but the last
    for (uint32_t mask = 0; mask < (1u << (T - 1)); ++mask) {
      G.clear();
      int run = 0;
      for (int w = 0; w < T; ++w) {
        ++run;
        if (w == T - 1 || ((mask >> w) & 1u)) {
          G.push_back(run);
          run = 0;
        }
      }
      if (prune && T > 1 && (G.front() > s1 || G.back() > sp)) continue;
      const double t = predict(G, duration_us, T, tiles, S, tile_bytes, c);
      bool better = best.empty() || t < best_t ||
                    (t == best_t && (G.size() < best.size() || (G.size() == best.size() && G < best)));
      if (better) {
        best = G;
        best_t = t;
      }
    }
    if (best.empty()) fail(FO_ERR_INVALID_ARG, "pruning left no candidate");
    for (size_t i = 0; i < best.size(); ++i) out_groups[i] = best[i];
    *out_num_groups = (int32_t)best.size();
    *predicted_us = best_t;
  });
}
