// a8 — iteration-time predictor: an event model of the fused hybrid-attention launch
// (include/niyama.h "a8"), its fit to measured launch times, and the
// a1 chunk choice (niyama_max_feasible_chunk).  The launch-shaping rules (split length,
// CTA split, queue orders) are the planner's own (internal.h), so the model sees the
// launch the kernel actually runs.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "internal.h"
#include "niyama.h"

using namespace niyama;

struct niyama_predictor {
  int hq = 0, hkv = 0, d = 0, elt = 0;
  int num_sms = NIYAMA_PRED_SMS;          // niyama_predictor_bind: the kv's device
  niyama_tuning tune = default_tuning();  // niyama_predictor_bind: the kv's tuning
  double theta[NIYAMA_NUM_PARAMS] = {0, 0, 0, 0, 0, 1, 1e-6, 0, 0, 2, 8e9, 1e-6, 7e12, 0, 1e11, 1};
  // full iteration (niyama_predictor_set_iteration): layers = 0 -> one attention launch
  int32_t layers = 0;
  std::vector<double> lin_t, lin_s;
  double it_c0 = 0, it_c1 = 0;
};

namespace {

niyama_status fail(niyama_status s, const std::string& m) { return set_error(s, m.c_str()); }

struct Run {  // `count` consecutive queue entries of equal size
  int64_t size;
  int64_t count;
};

// The launch as the planner builds it: independent of the model parameters.
struct Launch {
  double rows = 0, D = 0, sum_ctx = 0, units = 0;
  int32_t grid = 1, np = 0, wpc = 12, q = 0, small = 0, parts_target = 1;
  std::vector<int32_t> parts;  // split-K parts per slice (queue order)
  double bytes_per_token = 0;  // one kv head's K + V
  std::vector<Run> tiles;      // 128-key steps per tile, queue order
  std::vector<Run> pieces;     // tokens per decode unit, queue order
};

struct SliceOC {
  int32_t o, c;
};

void push_run(std::vector<Run>& v, int64_t size, int64_t count) {
  if (count <= 0) return;
  if (!v.empty() && v.back().size == size)
    v.back().count += count;
  else
    v.push_back(Run{size, count});
}

// Steps 1-3 of the model (niyama.h): tile queue, unit queue, grid and CTA split.
Launch build(const niyama_predictor& p, std::vector<SliceOC> slices, const int32_t* ctx, int64_t D) {
  Launch L;
  const int g = p.hq / p.hkv;
  const int64_t R = rows_per_tile(g);
  L.wpc = decode_streams(g, p.tune.decode_path);
  L.bytes_per_token = static_cast<double>(p.d) * 2.0 * p.elt;
  std::stable_sort(slices.begin(), slices.end(), [](const SliceOC& a, const SliceOC& b) {
    return static_cast<int64_t>(a.o) + a.c > static_cast<int64_t>(b.o) + b.c;
  });
  // q tiles per slice (steps of each, queue order); split-K parts are decided below
  std::vector<std::vector<int64_t>> qsteps(slices.size());
  int64_t q_tiles = 0, q_steps = 0;
  for (size_t si = 0; si < slices.size(); ++si) {
    const SliceOC& sl = slices[si];
    L.rows += sl.c;
    const int64_t nqt = ceil_div64(sl.c, R);
    for (int64_t qt = nqt - 1; qt >= 0; --qt) {
      const int64_t steps = ceil_div64(sl.o + std::min<int64_t>(sl.c, (qt + 1) * R), 128);
      qsteps[si].push_back(steps);
      q_tiles += p.hkv;
      q_steps += steps * p.hkv;
    }
  }
  int64_t sum_ctx = 0;
  int32_t max_ctx = 0;
  std::vector<int32_t> c(ctx, ctx + D);
  for (int32_t x : c) {
    sum_ctx += x;
    max_ctx = std::max(max_ctx, x);
  }
  int64_t n_units = 0;
  if (D > 0) {
    int32_t q = choose_split_len(sum_ctx, max_ctx, p.hkv, p.num_sms);
    if (p.tune.split_len > 0 && ceil_div64(max_ctx, p.tune.split_len) <= 4095) q = p.tune.split_len;
    const int32_t small = std::min<int32_t>(q, std::max<int32_t>(p.tune.tail_min, q / p.tune.tail_div));
    L.q = q;
    L.small = small;
    std::sort(c.begin(), c.end(), std::greater<int32_t>());  // the planner's queue: longest rows first
    std::vector<int32_t> tail;
    for (int32_t x : c) {
      const int64_t nf = ceil_div64(x, q) - 1;
      push_run(L.pieces, q, nf * p.hkv);  // full pieces, row by row
      for (int64_t k0 = nf * q; k0 < x; k0 += small) tail.push_back(static_cast<int32_t>(std::min<int64_t>(x, k0 + small) - k0));
      n_units += (nf + ceil_div64(x - nf * q, small)) * p.hkv;
    }
    std::sort(tail.begin(), tail.end(), std::greater<int32_t>());  // then the small pieces, longest first
    for (int32_t t : tail) push_run(L.pieces, t, p.hkv);
  }
  L.D = static_cast<double>(D);
  L.sum_ctx = static_cast<double>(sum_ctx);
  L.units = static_cast<double>(n_units);
  // split-K parts (internal.h, as the planner) and the work items in the kernel's order:
  // slices, q tiles (longest first), kv heads, parts
  const int32_t target = prefill_parts_target(q_tiles, n_units, q_steps + NIYAMA_TILE_SETUP_STEPS * q_tiles, sum_ctx,
                                              p.hkv, p.d, p.elt, g, p.num_sms, p.tune.decode_path, p.tune.prefill_split);
  L.parts_target = target;
  int64_t tile_cost = 0, n_tiles = 0;
  for (size_t si = 0; si < slices.size(); ++si) {
    const std::vector<int64_t>& qs = qsteps[si];
    if (qs.empty()) continue;
    const int32_t parts = target > 1 ? prefill_parts_of_slice(target, qs.back()) : 1;  // qs.back(): shortest tile
    L.parts.push_back(parts);
    for (int64_t nk : qs)
      for (int h = 0; h < p.hkv; ++h)
        for (int32_t part = 0; part < parts; ++part) {
          const int64_t steps = (part + 1) * nk / parts - part * nk / parts;
          push_run(L.tiles, steps, 1);
          tile_cost += steps + NIYAMA_TILE_SETUP_STEPS;
          ++n_tiles;
        }
  }
  const CtaSplit cs = cta_split(n_tiles, n_units, tile_cost, sum_ctx, p.hkv, p.d, p.elt, g, p.num_sms, p.tune.decode_path);
  L.grid = cs.grid;
  L.np = cs.prefill_ctas;
  if (p.tune.prefill_ctas > 0 && n_tiles > 0) L.np = std::min(p.tune.prefill_ctas, L.grid);
  if (p.tune.grid_cap > 0 && L.grid > p.tune.grid_cap) {
    L.grid = p.tune.grid_cap;
    L.np = std::min(L.np, L.grid);
  }
  return L;
}

// Ascending (time, count) buckets of interchangeable machines.
struct Buckets {
  std::vector<std::pair<double, int64_t>> b;
  void add(double t, int64_t n) {
    if (n <= 0) return;
    auto it = std::lower_bound(b.begin(), b.end(), t,
                               [](const std::pair<double, int64_t>& e, double v) { return e.first < v; });
    if (it != b.end() && it->first == t)
      it->second += n;
    else
      b.insert(it, {t, n});
  }
};

// Steps 4-5 (niyama.h): the launch as two coupled clocks.  Prefill: every busy
// prefill CTA advances on a common step clock S at 1/tau(t) steps per second,
// tau(t) = tau0 + tau_p P(t)/NSM + tau_d B(t)/W (P = prefill CTAs busy, B = decode
// warps busy, W = all warps of the grid); a tile of s steps taken at S = x ends at
// S = x + s + sigma (list scheduling: the queue's next tile goes to the CTA that frees
// first).  Decode (processor sharing): every busy warp streams at rate(t) =
// min(r_w, BW / B(t)) / (1 + gamma P(t)/NSM) on a common byte clock V; a unit of b
// bytes taken at V = v ends at V = v + b + u0 r_w; a free warp takes the queue's next
// unit.  The decode CTAs' warps start at 0, a prefill CTA's warps when the tile queue
// is empty and its last tile ended.  Returns the time the last tile or unit ends.
double simulate(const Launch& L, const double* nl) {
  const double tau0 = nl[0], tau_p = nl[1], tau_d = nl[2], sigma = nl[3], r_w = nl[4], u0 = nl[5], bw = nl[6],
               gamma = nl[7], r_cta = nl[8], sigma0 = nl[9];
  const double nsm = NIYAMA_PRED_SMS;
  const bool has_tiles = !L.tiles.empty() && L.np > 0;
  const double W = static_cast<double>(L.grid) * L.wpc;
  Buckets cta, busy;  // prefill CTAs: (end on S, count); decode warps: (end on V, count)
  double t = 0.0, S = 0.0, V = 0.0;
  int64_t P = 0, nbusy = 0;
  size_t trun = 0, prun = 0;
  int64_t tleft = has_tiles ? L.tiles[0].count : 0, pleft = L.pieces.empty() ? 0 : L.pieces[0].count;
  auto take_units = [&](int64_t n) {
    while (n > 0 && prun < L.pieces.size()) {
      const int64_t k = std::min(n, pleft);
      busy.add(V + static_cast<double>(L.pieces[prun].size) * L.bytes_per_token + u0 * r_w, k);
      nbusy += k;
      n -= k;
      if ((pleft -= k) == 0 && ++prun < L.pieces.size()) pleft = L.pieces[prun].count;
    }
  };
  auto take_tiles = [&](int64_t n) {  // n free prefill CTAs; returns how many found no tile
    while (n > 0 && trun < L.tiles.size()) {
      const int64_t k = std::min(n, tleft);
      cta.add(S + static_cast<double>(L.tiles[trun].size) + sigma, k);
      P += k;
      n -= k;
      if ((tleft -= k) == 0 && ++trun < L.tiles.size()) tleft = L.tiles[trun].count;
    }
    return n;
  };
  if (has_tiles) {  // a prefill CTA's first tile has setup sigma0 instead of sigma
    S = sigma0 - sigma;
    take_units(static_cast<int64_t>(L.grid - L.np) * L.wpc);
    take_units(take_tiles(L.np) * L.wpc);
    S = 0.0;
  }
  else {
    take_units(static_cast<int64_t>(L.grid) * L.wpc);
  }
  while (P > 0 || nbusy > 0) {
    const double tau = tau0 + tau_p * P / nsm + tau_d * nbusy / W;
    const double dec_ctas = std::max(1.0, static_cast<double>(L.grid - P));  // CTAs whose warps stream
    const double rate = nbusy > 0 ? std::min({r_w, bw / static_cast<double>(nbusy), r_cta * dec_ctas / static_cast<double>(nbusy)}) /
                                        (1.0 + gamma * P / nsm)
                                  : 0.0;
    const double dt_p = P > 0 ? (cta.b.front().first - S) * tau : std::numeric_limits<double>::infinity();
    const double dt_d = nbusy > 0 ? (busy.b.front().first - V) / rate : std::numeric_limits<double>::infinity();
    if (dt_p <= dt_d) {
      t += dt_p;
      if (nbusy > 0) V += dt_p * rate;
      S = cta.b.front().first;
      const int64_t k = cta.b.front().second;
      cta.b.erase(cta.b.begin());
      P -= k;
      take_units(take_tiles(k) * L.wpc);
    } else {
      t += dt_d;
      if (P > 0) S += dt_d / tau;
      V = busy.b.front().first;
      const int64_t k = busy.b.front().second;
      busy.b.erase(busy.b.begin());
      nbusy -= k;
      take_units(k);
    }
  }
  return t;
}

// Step 6: linear part.
constexpr int kLin = 6;
constexpr int kNl = NIYAMA_NUM_PARAMS - kLin;
void features(const Launch& L, double Tsim, double* f) {
  f[0] = 1.0;
  f[1] = L.rows + L.D;
  f[2] = L.D;
  f[3] = L.sum_ctx;
  f[4] = L.units;
  f[5] = Tsim;
}
double eval(const double* theta, const Launch& L) {
  double f[kLin];
  features(L, simulate(L, theta + kLin), f);
  double t = 0;
  for (int k = 0; k < kLin; ++k) t += theta[k] * f[k];
  return t;
}

bool parse_batch(const niyama_batch_desc* desc, std::vector<SliceOC>& sl) {
  if (!desc || desc->num_prefill < 0 || desc->num_decode < 0) return false;
  if (desc->num_prefill > 0 && (!desc->prefill_offset || !desc->prefill_len)) return false;
  if (desc->num_decode > 0 && !desc->decode_ctx) return false;
  for (int j = 0; j < desc->num_decode; ++j)
    if (desc->decode_ctx[j] < 1) return false;
  for (int i = 0; i < desc->num_prefill; ++i) {
    if (desc->prefill_offset[i] < 0 || desc->prefill_len[i] < 0) return false;
    if (desc->prefill_len[i] > 0) sl.push_back(SliceOC{desc->prefill_offset[i], desc->prefill_len[i]});
  }
  return true;
}

// ---------------------------------------------------------------- fit
// Least squares on the columns `cols` of A (m x n, row-major) by Householder QR.
bool lsq_subset(const std::vector<double>& A, int m, int n, const std::vector<double>& b, const std::vector<int>& cols,
                std::vector<double>& z) {
  const int k = static_cast<int>(cols.size());
  std::vector<double> M(static_cast<size_t>(m) * k), y(b);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < k; ++j) M[static_cast<size_t>(i) * k + j] = A[static_cast<size_t>(i) * n + cols[j]];
  for (int j = 0; j < k; ++j) {
    double norm = 0;
    for (int i = j; i < m; ++i) norm += M[static_cast<size_t>(i) * k + j] * M[static_cast<size_t>(i) * k + j];
    norm = std::sqrt(norm);
    if (norm == 0) return false;
    const double alpha = M[static_cast<size_t>(j) * k + j] > 0 ? -norm : norm;
    std::vector<double> v(m, 0.0);
    for (int i = j; i < m; ++i) v[i] = M[static_cast<size_t>(i) * k + j];
    v[j] -= alpha;
    double vn = 0;
    for (int i = j; i < m; ++i) vn += v[i] * v[i];
    if (vn == 0) continue;
    for (int jj = j; jj < k; ++jj) {
      double s = 0;
      for (int i = j; i < m; ++i) s += v[i] * M[static_cast<size_t>(i) * k + jj];
      s = 2 * s / vn;
      for (int i = j; i < m; ++i) M[static_cast<size_t>(i) * k + jj] -= s * v[i];
    }
    double s = 0;
    for (int i = j; i < m; ++i) s += v[i] * y[i];
    s = 2 * s / vn;
    for (int i = j; i < m; ++i) y[i] -= s * v[i];
  }
  z.assign(k, 0.0);
  for (int j = k - 1; j >= 0; --j) {
    double s = y[j];
    for (int jj = j + 1; jj < k; ++jj) s -= M[static_cast<size_t>(j) * k + jj] * z[jj];
    const double diag = M[static_cast<size_t>(j) * k + j];
    if (std::fabs(diag) < 1e-300) return false;
    z[j] = s / diag;
  }
  return true;
}

// Lawson-Hanson active-set NNLS: min ||A x - b||, x >= 0.
std::vector<double> nnls(const std::vector<double>& A, int m, int n, const std::vector<double>& b) {
  std::vector<double> x(n, 0.0);
  std::vector<bool> inP(n, false);
  double norm1 = 0;
  for (int j = 0; j < n; ++j) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += std::fabs(A[static_cast<size_t>(i) * n + j]);
    norm1 = std::max(norm1, s);
  }
  const double tol = 10.0 * std::max(m, n) * norm1 * std::numeric_limits<double>::epsilon();
  auto gradient = [&](std::vector<double>& w) {
    std::vector<double> r(b);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) r[i] -= A[static_cast<size_t>(i) * n + j] * x[j];
    w.assign(n, 0.0);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < m; ++i) w[j] += A[static_cast<size_t>(i) * n + j] * r[i];
  };
  std::vector<double> w;
  for (int outer = 0; outer < 3 * n + 10; ++outer) {
    gradient(w);
    int t = -1;
    double best = tol;
    for (int j = 0; j < n; ++j)
      if (!inP[j] && w[j] > best) best = w[j], t = j;
    if (t < 0) break;
    inP[t] = true;
    for (int inner = 0; inner < 3 * n + 10; ++inner) {
      std::vector<int> cols;
      for (int j = 0; j < n; ++j)
        if (inP[j]) cols.push_back(j);
      std::vector<double> zc;
      if (!lsq_subset(A, m, n, b, cols, zc)) {
        inP[cols.back()] = false;
        break;
      }
      std::vector<double> z(n, 0.0);
      for (size_t k = 0; k < cols.size(); ++k) z[cols[k]] = zc[k];
      bool allpos = true;
      for (int j : cols)
        if (z[j] <= 0) allpos = false;
      if (allpos) {
        x = z;
        break;
      }
      double alpha = 2.0;
      for (int j : cols)
        if (z[j] <= 0) alpha = std::min(alpha, x[j] / (x[j] - z[j]));
      for (int j = 0; j < n; ++j) x[j] += alpha * (z[j] - x[j]);
      for (int j : cols)
        if (x[j] <= tol) {
          x[j] = 0;
          inP[j] = false;
        }
    }
  }
  return x;
}

// Given the nonlinear parameters: the launch simulations of every sample (in
// parallel), the linear weights theta[0..4] >= 0 by NNLS on relative residuals with
// the simulation's weight theta[5] fixed at 1, and the sum of squared relative errors.
double fit_linear(const std::vector<Launch>& L, const std::vector<double>& t, const double* nl, double* lin_out) {
  const int m = static_cast<int>(L.size());
  std::vector<double> Tsim(m);
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  const int nth = m >= 64 ? static_cast<int>(hw) : 1;
  std::vector<std::thread> th;
  for (int k = 0; k < nth; ++k)
    th.emplace_back([&, k] {
      for (int i = k; i < m; i += nth) Tsim[i] = simulate(L[i], nl);
    });
  for (auto& x : th) x.join();
  const int n = kLin - 1;
  std::vector<double> A(static_cast<size_t>(m) * n), b(m);
  double colmax[kLin] = {0};
  for (int i = 0; i < m; ++i) {
    double f[kLin];
    features(L[i], Tsim[i], f);
    for (int k = 0; k < n; ++k) {
      A[static_cast<size_t>(i) * n + k] = f[k] / t[i];
      colmax[k] = std::max(colmax[k], std::fabs(A[static_cast<size_t>(i) * n + k]));
    }
    b[i] = 1.0 - Tsim[i] / t[i];
  }
  for (int k = 0; k < n; ++k) {
    if (colmax[k] == 0) colmax[k] = 1;
    for (int i = 0; i < m; ++i) A[static_cast<size_t>(i) * n + k] /= colmax[k];
  }
  const std::vector<double> z = nnls(A, m, n, b);
  for (int k = 0; k < n; ++k) lin_out[k] = z[k] / colmax[k];
  lin_out[n] = 1.0;
  double s = 0;
  for (int i = 0; i < m; ++i) {
    double f[kLin];
    features(L[i], Tsim[i], f);
    double tt = 0;
    for (int k = 0; k < kLin; ++k) tt += lin_out[k] * f[k];
    const double e = tt / t[i] - 1.0;
    s += e * e;
  }
  return s;
}

// Nonlinear parameters live in log space inside these bounds (s, s, s, steps, B/s, s, B/s, 1).
constexpr double kLo[kNl] = {1e-8, 1e-10, 1e-10, 1e-3, 1e8, 1e-9, 1e11, 1e-4, 1e9, 1e-3};
constexpr double kHi[kNl] = {1e-4, 1e-4, 1e-4, 1e3, 1e12, 1e-3, 1e14, 1e2, 1e13, 1e3};
constexpr double kStart[kNl] = {0.8e-6, 0.1e-6, 0.15e-6, 4.0, 30e9, 0.2e-6, 9.0e12, 0.2, 100e9, 5.0};

void from_log(const double* x, double* nl) {
  for (int k = 0; k < kNl; ++k) nl[k] = std::exp(std::min(std::log(kHi[k]), std::max(std::log(kLo[k]), x[k])));
}

// Nelder-Mead (standard coefficients 1, 2, 0.5, 0.5) on the log-parameters.
void nelder_mead(const std::vector<Launch>& L, const std::vector<double>& t, double* x0, int max_evals) {
  const int n = kNl;
  std::vector<std::vector<double>> s(n + 1, std::vector<double>(x0, x0 + n));
  std::vector<double> fv(n + 1);
  double lin[kLin], nl[kNl];
  auto f = [&](const std::vector<double>& x) {
    from_log(x.data(), nl);
    return fit_linear(L, t, nl, lin);
  };
  for (int k = 0; k < n; ++k) s[k + 1][k] += 0.5;  // initial simplex: factor e^0.5 per parameter
  for (int k = 0; k <= n; ++k) fv[k] = f(s[k]);
  int evals = n + 1;
  while (evals < max_evals) {
    std::vector<int> idx(n + 1);
    for (int k = 0; k <= n; ++k) idx[k] = k;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return fv[a] < fv[b]; });
    const int best = idx[0], worst = idx[n], second = idx[n - 1];
    if (std::fabs(fv[worst] - fv[best]) <= 1e-10 * std::max(1e-30, std::fabs(fv[best]))) break;
    std::vector<double> c(n, 0.0);
    for (int k = 0; k < n; ++k)
      for (int j = 0; j < n; ++j) c[j] += s[idx[k]][j] / n;
    auto along = [&](double a) {
      std::vector<double> x(n);
      for (int j = 0; j < n; ++j) x[j] = c[j] + a * (s[worst][j] - c[j]);
      return x;
    };
    std::vector<double> xr = along(-1.0);
    const double fr = f(xr);
    ++evals;
    if (fr < fv[best]) {
      std::vector<double> xe = along(-2.0);
      const double fe = f(xe);
      ++evals;
      if (fe < fr) s[worst] = xe, fv[worst] = fe;
      else s[worst] = xr, fv[worst] = fr;
    } else if (fr < fv[second]) {
      s[worst] = xr, fv[worst] = fr;
    } else {
      std::vector<double> xc = fr < fv[worst] ? along(-0.5) : along(0.5);
      const double fc = f(xc);
      ++evals;
      if (fc < std::min(fr, fv[worst])) {
        s[worst] = xc, fv[worst] = fc;
      } else {
        for (int k = 1; k <= n; ++k) {
          for (int j = 0; j < n; ++j) s[idx[k]][j] = s[best][j] + 0.5 * (s[idx[k]][j] - s[best][j]);
          fv[idx[k]] = f(s[idx[k]]);
          ++evals;
        }
      }
    }
  }
  int b = 0;
  for (int k = 1; k <= n; ++k)
    if (fv[k] < fv[b]) b = k;
  for (int j = 0; j < n; ++j) x0[j] = s[b][j];
}

niyama_status pred_shape(const niyama_kv_config* s, niyama_predictor* p) {
  if (!s) return fail(NIYAMA_EINVAL, "shape is NULL");
  if (s->world_size < 1 || s->num_kv_heads < 1 || s->num_q_heads < 1 || s->head_dim < 1 ||
      s->num_kv_heads % s->world_size || s->num_q_heads % s->world_size || s->num_q_heads % s->num_kv_heads)
    return fail(NIYAMA_EINVAL, "predictor shape");
  p->hq = s->num_q_heads / s->world_size;
  p->hkv = s->num_kv_heads / s->world_size;
  p->d = s->head_dim;
  p->elt = s->dtype == NIYAMA_BF16 ? 2 : 4;
  return NIYAMA_OK;
}

bool feasible(double t, double slack) { return t <= slack + 1e-12 * std::max(1.0, std::fabs(slack)); }

niyama_status fit_launches(niyama_predictor& p, const std::vector<Launch>& L, const std::vector<double>& t,
                           const niyama_fit_options* opt, niyama_predictor** out) {
  double x[kNl];
  for (int k = 0; k < kNl; ++k) x[k] = std::log(opt && opt->start ? opt->start[kLin + k] : kStart[k]);
  const int evals = opt && opt->max_evals > 0 ? opt->max_evals : 1200;
  const int stride = opt && opt->subsample > 1 ? opt->subsample : 1;
  std::vector<Launch> Ls;
  std::vector<double> ts;
  for (size_t i = 0; i < L.size(); i += stride) Ls.push_back(L[i]), ts.push_back(t[i]);
  nelder_mead(Ls, ts, x, evals);
  nelder_mead(Ls, ts, x, evals / 2);  // restart from the best vertex (escapes a collapsed simplex)
  double nl[kNl], lin[kLin];
  from_log(x, nl);
  fit_linear(L, t, nl, lin);
  auto* res = new niyama_predictor(p);
  for (int k = 0; k < kLin; ++k) res->theta[k] = lin[k];
  for (int k = 0; k < kNl; ++k) res->theta[kLin + k] = nl[k];
  *out = res;
  return NIYAMA_OK;
}

}  // namespace

extern "C" niyama_status niyama_predictor_fit_batches(const niyama_kv_config* shape, const niyama_batch_desc* batches,
                                                      const double* seconds, int32_t n, const niyama_fit_options* opt,
                                                      niyama_predictor** out) {
  if (!out) return fail(NIYAMA_EINVAL, "out is NULL");
  *out = nullptr;
  if (!batches || !seconds || n < 1) return fail(NIYAMA_EINVAL, "no samples");
  niyama_predictor p;
  niyama_status st = pred_shape(shape, &p);
  if (st != NIYAMA_OK) return st;
  if (opt && opt->start) {
    for (int k = 0; k < NIYAMA_NUM_PARAMS; ++k)
      if (!std::isfinite(opt->start[k]) || (k >= kLin && !(opt->start[k] > 0)))
        return fail(NIYAMA_EINVAL, "fit options: start");
  }
  std::vector<Launch> L;
  std::vector<double> t;
  for (int i = 0; i < n; ++i) {
    std::vector<SliceOC> sl;
    if (!(seconds[i] > 0) || !std::isfinite(seconds[i]) || !parse_batch(&batches[i], sl))
      return fail(NIYAMA_EINVAL, "sample " + std::to_string(i) + " is invalid");
    L.push_back(build(p, std::move(sl), batches[i].decode_ctx, batches[i].num_decode));
    t.push_back(seconds[i]);
  }
  return fit_launches(p, L, t, opt, out);
}

extern "C" niyama_status niyama_predictor_fit(const niyama_kv_config* shape, const niyama_sample* samples, int32_t n,
                                              niyama_predictor** out) {
  if (!out) return fail(NIYAMA_EINVAL, "out is NULL");
  *out = nullptr;
  if (!samples || n < 1) return fail(NIYAMA_EINVAL, "no samples");
  niyama_predictor p;
  niyama_status st = pred_shape(shape, &p);
  if (st != NIYAMA_OK) return st;
  std::vector<Launch> L;
  std::vector<double> t;
  for (int i = 0; i < n; ++i) {
    const niyama_sample& s = samples[i];
    if (!(s.seconds > 0) || !std::isfinite(s.seconds) || s.chunk_len < 0 || s.chunk_offset < 0 || s.num_decode < 0 ||
        s.sum_ctx < s.num_decode || (s.num_decode == 0 && s.sum_ctx != 0) ||
        s.sum_ctx / std::max(1, s.num_decode) >= (int64_t(1) << 30))
      return fail(NIYAMA_EINVAL, "sample " + std::to_string(i) + " is invalid");
    std::vector<SliceOC> sl;
    if (s.chunk_len > 0) sl.push_back(SliceOC{s.chunk_offset, s.chunk_len});
    std::vector<int32_t> ctx(s.num_decode);
    if (s.num_decode > 0) {
      const int64_t base = s.sum_ctx / s.num_decode, rem = s.sum_ctx % s.num_decode;
      for (int32_t j = 0; j < s.num_decode; ++j) ctx[j] = static_cast<int32_t>(base + (j < rem ? 1 : 0));
    }
    L.push_back(build(p, std::move(sl), ctx.data(), s.num_decode));
    t.push_back(s.seconds);
  }
  return fit_launches(p, L, t, nullptr, out);
}

extern "C" niyama_status niyama_predictor_from_params(const niyama_kv_config* shape, const double* theta,
                                                      niyama_predictor** out) {
  if (!out || !theta) return fail(NIYAMA_EINVAL, "out/theta is NULL");
  *out = nullptr;
  niyama_predictor p;
  niyama_status st = pred_shape(shape, &p);
  if (st != NIYAMA_OK) return st;
  for (int k = 0; k < NIYAMA_NUM_PARAMS; ++k) {
    const bool ok = std::isfinite(theta[k]) && (k < kLin ? theta[k] >= 0 : theta[k] > 0);
    if (!ok) return fail(NIYAMA_EINVAL, "theta: linear part finite and >= 0, event-model part finite and > 0");
    p.theta[k] = theta[k];
  }
  *out = new niyama_predictor(p);
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_predictor_params(const niyama_predictor* p, double* theta_out) {
  if (!p || !theta_out) return fail(NIYAMA_EINVAL, "p/out is NULL");
  std::memcpy(theta_out, p->theta, sizeof(p->theta));
  return NIYAMA_OK;
}

namespace {
double lin_table(const niyama_predictor& p, double T) {
  const std::vector<double>& x = p.lin_t;
  const std::vector<double>& y = p.lin_s;
  const size_t n = x.size();
  size_t i = 1;
  while (i + 1 < n && x[i] < T) ++i;  // segment [i-1, i] (the first / last one extrapolates)
  return y[i - 1] + (y[i] - y[i - 1]) * (T - x[i - 1]) / (x[i] - x[i - 1]);
}
// One attention launch or, with layers > 0, the full iteration.
double total(const niyama_predictor& p, const Launch& L) {
  const double a = eval(p.theta, L);
  if (p.layers <= 0) return a;
  const double T = L.rows + L.D;
  return p.it_c0 + p.it_c1 * T + lin_table(p, T) + p.layers * a;
}
}  // namespace

extern "C" double niyama_predict_iter_time(const niyama_predictor* p, const niyama_batch_desc* desc) {
  std::vector<SliceOC> sl;
  if (!p || !parse_batch(desc, sl)) return -1.0;
  return total(*p, build(*p, std::move(sl), desc->decode_ctx, desc->num_decode));
}

extern "C" niyama_status niyama_predictor_set_iteration(niyama_predictor* p, int32_t layers, const int32_t* tokens,
                                                        const double* seconds, int32_t n, double c0, double c1) {
  if (!p) return fail(NIYAMA_EINVAL, "predictor is NULL");
  if (layers < 0) return fail(NIYAMA_EINVAL, "layers < 0");
  if (layers == 0) {
    p->layers = 0;
    p->lin_t.clear();
    p->lin_s.clear();
    p->it_c0 = p->it_c1 = 0;
    return NIYAMA_OK;
  }
  if (!tokens || !seconds || n < 2) return fail(NIYAMA_EINVAL, "linear table needs >= 2 points");
  for (int i = 0; i < n; ++i)
    if (tokens[i] <= 0 || (i > 0 && tokens[i] <= tokens[i - 1]) || !(seconds[i] >= 0) || !std::isfinite(seconds[i]))
      return fail(NIYAMA_EINVAL, "linear table: tokens ascending and > 0, seconds >= 0");
  if (!std::isfinite(c0) || !std::isfinite(c1)) return fail(NIYAMA_EINVAL, "c0/c1");
  p->layers = layers;
  p->lin_t.assign(tokens, tokens + n);
  p->lin_s.assign(seconds, seconds + n);
  p->it_c0 = c0;
  p->it_c1 = c1;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_predictor_fit_iteration(niyama_predictor* p, const niyama_batch_desc* batches,
                                                        const double* seconds, int32_t n) {
  if (!p || !batches || !seconds || n < 2) return fail(NIYAMA_EINVAL, "NULL argument or n < 2");
  if (p->layers <= 0) return fail(NIYAMA_ESTATE, "set the iteration table first");
  // min sum ((c0 + c1 T + r_i) / t_i - 1)^2 over (c0, c1), r_i = lin(T_i) + layers * t_hat_i
  double a11 = 0, a12 = 0, a22 = 0, b1 = 0, b2 = 0;
  for (int i = 0; i < n; ++i) {
    std::vector<SliceOC> sl;
    if (!(seconds[i] > 0) || !parse_batch(&batches[i], sl)) return fail(NIYAMA_EINVAL, "sample " + std::to_string(i));
    const Launch L = build(*p, std::move(sl), batches[i].decode_ctx, batches[i].num_decode);
    const double T = L.rows + L.D, t = seconds[i];
    const double r = lin_table(*p, T) + p->layers * eval(p->theta, L);
    const double u = 1.0 / t, v = T / t, y = 1.0 - r / t;
    a11 += u * u, a12 += u * v, a22 += v * v, b1 += u * y, b2 += v * y;
  }
  const double det = a11 * a22 - a12 * a12;
  if (!(std::fabs(det) > 0)) return fail(NIYAMA_EINVAL, "degenerate samples (all T equal)");
  p->it_c0 = (b1 * a22 - b2 * a12) / det;
  p->it_c1 = (a11 * b2 - a12 * b1) / det;
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_predict_detail(const niyama_predictor* p, const niyama_batch_desc* desc,
                                               niyama_predict_info* out) {
  std::vector<SliceOC> sl;
  if (!p || !out) return fail(NIYAMA_EINVAL, "NULL argument");
  if (!parse_batch(desc, sl)) return fail(NIYAMA_EINVAL, "batch descriptor");
  const Launch L = build(*p, std::move(sl), desc->decode_ctx, desc->num_decode);
  out->grid = L.grid;
  out->prefill_ctas = L.np;
  out->split_len = L.q;
  out->small_piece = L.small;
  out->warps_per_cta = L.wpc;
  out->prefill_parts_target = L.parts_target;
  out->num_units = static_cast<int64_t>(L.units);
  out->sim_seconds = simulate(L, p->theta + kLin);
  out->seconds = total(*p, L);
  return NIYAMA_OK;
}

extern "C" niyama_status niyama_max_feasible_chunk(const niyama_predictor* p, const niyama_batch_desc* decodes_only,
                                                   int32_t chunk_offset, int32_t prefill_remaining, double slack_s,
                                                   int32_t max_chunk, int32_t* chunk_out, int32_t* infeasible_out) {
  if (!p || !decodes_only || !chunk_out || !infeasible_out) return fail(NIYAMA_EINVAL, "NULL argument");
  if (chunk_offset < 0 || max_chunk < 0 || std::isnan(slack_s)) return fail(NIYAMA_EINVAL, "chunk_offset/max_chunk/slack");
  if (decodes_only->num_decode < 0 || (decodes_only->num_decode > 0 && !decodes_only->decode_ctx))
    return fail(NIYAMA_EINVAL, "decode arrays");
  for (int j = 0; j < decodes_only->num_decode; ++j)
    if (decodes_only->decode_ctx[j] < 1) return fail(NIYAMA_EINVAL, "decode_ctx < 1");
  auto t_of = [&](int32_t C) {
    std::vector<SliceOC> sl;
    if (C > 0) sl.push_back(SliceOC{chunk_offset, C});
    return total(*p, build(*p, std::move(sl), decodes_only->decode_ctx, decodes_only->num_decode));
  };
  const int32_t cap = std::max(0, std::min(max_chunk, prefill_remaining));
  *infeasible_out = 0;
  if (!feasible(t_of(0), slack_s)) {
    *chunk_out = 0;
    *infeasible_out = 1;
    return NIYAMA_OK;
  }
  if (feasible(t_of(cap), slack_s)) {
    *chunk_out = cap;
    return NIYAMA_OK;
  }
  int32_t lo = 0, hi = cap;  // t_of(lo) feasible, t_of(hi) not
  while (hi - lo > 1) {
    const int32_t mid = lo + (hi - lo) / 2;
    if (feasible(t_of(mid), slack_s))
      lo = mid;
    else
      hi = mid;
  }
  *chunk_out = lo;
  return NIYAMA_OK;
}

extern "C" void niyama_predictor_destroy(niyama_predictor* p) { delete p; }

extern "C" niyama_status niyama_predictor_bind(niyama_predictor* p, const niyama_kv* kv) {
  if (!p || !kv) return fail(NIYAMA_EINVAL, "predictor/kv is NULL");
  KvModel m{};
  kv_model(kv, &m);
  if (p->hq != m.hq || p->hkv != m.hkv || p->d != m.d || p->elt != m.elt)
    return fail(NIYAMA_EINVAL, "predictor shape differs from the kv's local shape");
  p->num_sms = m.num_sms;
  p->tune = m.tune;
  return NIYAMA_OK;
}
