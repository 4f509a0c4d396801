// placement.cpp -- pi_place_ilp: the paper's neuron-placement ILP (Eqs. 1-8), solved
// exactly on the host (include/pi.h; oracle: oracle/placement.py).
//
// Two units, fast and slow.  Each layer's neurons are ordered by (-f_i, i) and grouped into
// batches of `granule` similar-impact neurons; a batch is placed whole.  Maximise the
// impact on the fast unit (Eq. 2, v_i = f_i by Eq. 1) subject to: every batch on one unit (Eq. 3),
// the fast unit's capacity (Eq. 6, strict), and per layer either nothing on the fast unit or at
// least C_l neurons, C_l the smallest count with C_l T_l^fast + T_sync <= C_l T_l^slow (Eqs. 4, 5,
// 7, 8; reading R22).
//
// Within a layer all full batches cost the same memory, so for any number j of fast full batches
// the best choice is the j most impactful ones (the first j in (-f, i) order); a ragged last
// batch (m % granule != 0) is a separate item, taken or not.  The ILP is therefore a group
// knapsack over layers -- per layer one option (j, last batch or not) with a count of 0 or >= C_l
// -- solved by dynamic programming over capacity in units of the gcd of the batch sizes (exact;
// no LP relaxation, no heuristic).  Ties go to fewer fast bytes, then to lower layers.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <vector>

#include "../../include/pi.h"

extern pi_status pi_set_error(pi_status st, const char *msg);

static int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

extern "C" pi_status pi_place_ilp(const float *freq, int32_t n_layers, int32_t m, const double *neuron_bytes,
                                  int32_t granule, double mcap_fast, double bw_fast, double bw_slow, double t_sync,
                                  uint8_t *fast, int32_t *fast_count, double *objective) {
  char buf[256];
  pi_set_error(PI_OK, "");
  if (!freq || !neuron_bytes || !fast || !fast_count || !objective)
    return pi_set_error(PI_ERR_INVALID_ARGUMENT, "pi_place_ilp: NULL argument");
  if (n_layers < 1 || m < 1 || granule < 1 || !(bw_fast > 0) || !(bw_slow > 0) || !(t_sync >= 0) ||
      !(mcap_fast >= 0) || std::isnan(mcap_fast)) {
    snprintf(buf, sizeof buf, "pi_place_ilp: bad sizes or parameters (L=%d m=%d granule=%d)", n_layers, m, granule);
    return pi_set_error(PI_ERR_INVALID_ARGUMENT, buf);
  }
  const int L = n_layers;
  std::vector<int64_t> nbytes(L);
  for (int l = 0; l < L; ++l) {
    const double b = neuron_bytes[l];
    if (!(b >= 1) || b != std::floor(b) || b > 1e15)
      return pi_set_error(PI_ERR_INVALID_ARGUMENT, "pi_place_ilp: neuron_bytes must be positive integers");
    nbytes[l] = (int64_t)b;
  }
  for (int64_t i = 0; i < (int64_t)L * m; ++i)
    if (!std::isfinite(freq[i]) || freq[i] < 0.f)
      return pi_set_error(PI_ERR_INVALID_ARGUMENT, "pi_place_ilp: freq must be finite and >= 0");

  // batches per layer in (-f, i) order: nfull full batches, then a ragged one of `rem` neurons
  const int nfull = m / granule, rem = m - nfull * granule;
  std::vector<std::vector<int32_t>> order(L, std::vector<int32_t>(m));
  std::vector<std::vector<double>> pval(L, std::vector<double>(nfull + 1, 0.0));   // prefix of full batches
  std::vector<double> vrem(L, 0.0);
  int64_t unit = 0;
  for (int l = 0; l < L; ++l) {
    const float *f = freq + (int64_t)l * m;
    std::iota(order[l].begin(), order[l].end(), 0);
    std::sort(order[l].begin(), order[l].end(), [&](int32_t a, int32_t b) {
      if (f[a] != f[b]) return f[a] > f[b];
      return a < b;
    });
    for (int k = 0; k < nfull; ++k) {
      double v = 0.0;
      for (int q = k * granule; q < (k + 1) * granule; ++q) v += (double)f[order[l][q]];
      pval[l][k + 1] = pval[l][k] + v;
    }
    for (int q = nfull * granule; q < m; ++q) vrem[l] += (double)f[order[l][q]];
    if (nfull) unit = gcd64(unit, (int64_t)granule * nbytes[l]);
    if (rem) unit = gcd64(unit, (int64_t)rem * nbytes[l]);
  }
  // Eq. 6 (strict): sum of fast bytes < mcap_fast  <=>  units <= ceil(mcap / unit) - 1
  // (capacity beyond all batches' bytes changes nothing: clamp to the total)
  int64_t total_units = 0;
  for (int l = 0; l < L; ++l) total_units += (int64_t)m * nbytes[l] / unit;
  const double cap_units_d = std::ceil(mcap_fast / (double)unit) - 1.0;
  const int64_t cap = cap_units_d < 0 ? -1 : (int64_t)std::min(cap_units_d, (double)total_units);
  std::vector<int64_t> cmin(L);   // Eqs. 4-5: smallest C_l with C_l T_fast + T_sync <= C_l T_slow; -1: none
  for (int l = 0; l < L; ++l) {
    const double tf = (double)nbytes[l] / bw_fast, ts = (double)nbytes[l] / bw_slow;
    int64_t c = -1;
    if (ts > tf) {
      c = (int64_t)std::ceil(t_sync / (ts - tf) - 1e-12);
      if (c < 0) c = 0;
      while ((double)c * tf + t_sync > (double)c * ts) ++c;
    }
    cmin[l] = c;
  }
  const int64_t cells = (int64_t)L * (std::max<int64_t>(cap, 0) + 1);
  if (cells > 64ll * 1000 * 1000)
    return pi_set_error(PI_ERR_UNSUPPORTED, "pi_place_ilp: capacity / batch-size ratio too large for the exact DP");
  std::fill(fast, fast + (int64_t)L * m, (uint8_t)0);
  for (int l = 0; l < L; ++l) fast_count[l] = 0;
  *objective = 0.0;
  if (cap < 0) return PI_OK;   // nothing fits (Eq. 6 is strict)

  // option o of a layer: j = o >> 1 full batches, plus the ragged batch if (o & 1)
  const int nopt = 2 * (nfull + 1);
  std::vector<double> best(cap + 1, 0.0), nb(cap + 1);
  std::vector<int32_t> choice((size_t)L * (cap + 1), 0);
  for (int l = 0; l < L; ++l) {
    for (int64_t u = 0; u <= cap; ++u) {
      double bv = best[u];   // count 0 (y_l = 0, Eqs. 7-8)
      int bo = 0;
      for (int o = 1; o < nopt; ++o) {
        const int j = o >> 1, p = o & 1;
        if (p && !rem) continue;
        const int64_t cnt = (int64_t)j * granule + (p ? rem : 0);
        if (cnt == 0 || cmin[l] < 0 || cnt < cmin[l]) continue;   // Eqs. 4, 7
        const int64_t cost = cnt * nbytes[l] / unit;
        if (cost > u) continue;
        const double v = best[u - cost] + pval[l][j] + (p ? vrem[l] : 0.0);
        if (v > bv + 1e-12 * std::max(1.0, std::fabs(v))) {
          bv = v;
          bo = o;
        }
      }
      nb[u] = bv;
      choice[(size_t)l * (cap + 1) + u] = bo;
    }
    best.swap(nb);
  }
  // best[u] is non-decreasing in u (capacity is an upper bound): read the optimum at u = cap and
  // walk the choices back, layer L-1 down to 0
  int64_t u = cap;
  for (int l = L - 1; l >= 0; --l) {
    const int o = choice[(size_t)l * (cap + 1) + u];
    if (o > 0) {
      const int j = o >> 1, p = o & 1;
      for (int64_t q = 0; q < (int64_t)j * granule; ++q) fast[(int64_t)l * m + order[l][q]] = 1;
      if (p)
        for (int q = nfull * granule; q < m; ++q) fast[(int64_t)l * m + order[l][q]] = 1;
      const int64_t cnt = (int64_t)j * granule + (p ? rem : 0);
      fast_count[l] = (int32_t)cnt;
      u -= cnt * nbytes[l] / unit;
    }
  }
  *objective = best[cap];
  return PI_OK;
}
