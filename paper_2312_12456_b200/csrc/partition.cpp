// partition.cpp -- pi_partition: host-side neuron -> GPU placement (include/pi.h).
//
// The paper solves an ILP over GPU/CPU placement (Eqs. 2-8) with
// 64 similar-impact neurons grouped into one decision, impact
// v_i = f_i (Eq. 1).  For G identical GPUs (reading R15) the
// objective becomes: each neuron on exactly one GPU (Eq. 3), equal counts
// (Eq. 6, equal capacities), minimal maximum expected active mass.  Solved by
// LPT under a cardinality cap:
//   order by (-f_i, i); cut into runs of `granule`; run load = sum f (double, run
//   order); runs in order go to the least-loaded shard with room (ties: lowest).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/pi.h"

// error state lives in pi_api.cu
extern pi_status pi_set_error(pi_status st, const char *msg);

extern "C" pi_status pi_partition(const float *freq, int32_t m, int32_t n_shards, int32_t granule,
                                  int32_t *owner, int32_t *shard_ids, int32_t *shard_offsets) {
  char buf[256];
  pi_set_error(PI_OK, "");
  if (!freq || !owner || !shard_ids || !shard_offsets)
    return pi_set_error(PI_ERR_INVALID_ARGUMENT, "pi_partition: NULL argument");
  if (n_shards < 1 || granule < 1 || m < 1) {
    snprintf(buf, sizeof buf, "pi_partition: m=%d n_shards=%d granule=%d must be >= 1", m, n_shards, granule);
    return pi_set_error(PI_ERR_INVALID_ARGUMENT, buf);
  }
  if ((int64_t)m % ((int64_t)granule * n_shards) != 0) {
    snprintf(buf, sizeof buf, "pi_partition: m=%d not divisible by granule*n_shards=%lld", m,
             (long long)granule * n_shards);
    return pi_set_error(PI_ERR_SHAPE, buf);
  }
  std::vector<double> f(m);
  for (int i = 0; i < m; ++i) {
    const float v = freq[i];
    if (!std::isfinite(v) || v < 0.f) {
      snprintf(buf, sizeof buf, "pi_partition: freq[%d]=%g must be finite and >= 0", i, (double)v);
      return pi_set_error(PI_ERR_INVALID_ARGUMENT, buf);
    }
    f[i] = (double)v;
  }
  std::vector<int32_t> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    if (f[a] != f[b]) return f[a] > f[b];
    return a < b;
  });
  const int n_runs = m / granule;
  const int cap = n_runs / n_shards;
  std::vector<double> load(n_shards, 0.0);
  std::vector<int> count(n_shards, 0);
  for (int k = 0; k < n_runs; ++k) {
    double rl = 0.0;
    for (int q = 0; q < granule; ++q) rl += f[order[(size_t)k * granule + q]];
    int best = -1;
    for (int g = 0; g < n_shards; ++g) {
      if (count[g] >= cap) continue;
      if (best < 0 || load[g] < load[best]) best = g;
    }
    load[best] += rl;
    count[best] += 1;
    for (int q = 0; q < granule; ++q) owner[order[(size_t)k * granule + q]] = best;
  }
  int pos = 0;
  shard_offsets[0] = 0;
  for (int g = 0; g < n_shards; ++g) {
    for (int i = 0; i < m; ++i)
      if (owner[i] == g) shard_ids[pos++] = i;
    shard_offsets[g + 1] = pos;
  }
  return PI_OK;
}
