// pi_api.cu -- libpi's C ABI (include/pi.h): validation, layer handles, workspace,
// and dispatch of the sm_100a kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/pi.h"
#include "fused_host.h"
#include "launch.h"

using namespace pi;

// ---------------------------------------------------------------------------
// error state
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static pi_status fail(pi_status st, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

pi_status pi_set_error(pi_status st, const char *msg) {
  g_err = msg;
  return st;
}

#define PI_CUDA(call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? PI_ERR_OUT_OF_MEMORY : PI_ERR_CUDA, \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define PI_TRY(expr)                \
  do {                              \
    pi_status s_ = (expr);          \
    if (s_ != PI_OK) return s_;     \
  } while (0)

// ---------------------------------------------------------------------------
// the handle
// ---------------------------------------------------------------------------
struct pi_layer {
  int device = 0;
  int num_sms = 148;
  int layer_id = 0;
  int d = 0, m_local = 0, r = 0, words = 0, max_batch = 1;
  pi_dtype dtype = PI_DT_BF16;
  pi_ffn_format ffn = PI_FFN_16;
  int64_t rec_q4 = 0;   // PI_FFN_Q4: bytes of one neuron record (d/2 codes + d/32 fp16 scales, 16-B padded)
  pi_act act = PI_ACT_RELU;
  pi_pred_act pred_act = PI_PRED_RELU;
  uint32_t flags = 0;
  float threshold = 0.f;
  // library-owned weights (16-bit elements)
  void *w_up = nullptr;    // [m_local, d] or interleaved [m_local, 2, d] (gate, up)
  void *w_down = nullptr;  // [m_local, d] (transposed)
  void *b_up = nullptr, *b_down = nullptr;
  void *p_w1 = nullptr, *p_b1 = nullptr, *p_w2 = nullptr, *p_b2 = nullptr;
  // workspace
  float *g = nullptr;         // [max_batch, r]
  float *scale = nullptr;     // [max_batch]
  float *h = nullptr;         // [max_batch, m_local]
  float *partial = nullptr;   // [S, max_batch, d]
  float *upart = nullptr;     // [ceil(d/256), m_local, 2, min(max_batch, 8)] (k_up_xs, max_batch >= 6)
  unsigned *tickets = nullptr;  // [tiles]
  uint32_t *mask = nullptr;   // [max_batch, words]
  int32_t *ids = nullptr;     // [m_local]
  int32_t *n_active = nullptr;
  float *xbuf = nullptr, *ybuf = nullptr;  // [max_batch, d] each (stack ping-pong)
  float *hx = nullptr, *hy = nullptr;      // [max_batch, d] each (host-buffer entry points)
  // batched tensor-core path (max_batch > 8): activation splits, partials, tickets (tc.cuh)
  uint16_t *x3 = nullptr, *h3 = nullptr;
  float *partial_tc = nullptr;
  unsigned *tickets_tc = nullptr;
  int S_tc = 0;
  int32_t *hot_ids = nullptr;              // [n_hot] local ids of hot neurons, hottest first
  uint32_t *hot_words = nullptr;           // [words] bitmap of the first hot_cap of them (prefetched set)
  int n_hot = 0, hot_cap = 0;
  int32_t *spec_ids = nullptr;             // [n_spec] speculative hot prefix, hottest first
  uint32_t *spec_words = nullptr;          // [words] bitmap of the speculative neurons
  int n_spec = 0;
  FusedWork fw{};             // fused-kernel workspace
  int tiles = 0, S = 0;
  int64_t weight_bytes = 0, ws_bytes = 0;
  std::vector<void *> allocs;
};

static pi_status dev_alloc(pi_layer *L, void **p, size_t bytes, bool weight) {
  if (bytes == 0) bytes = 16;
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(PI_ERR_OUT_OF_MEMORY, "layer %d: cudaMalloc(%zu) failed: %s", L->layer_id, bytes,
                cudaGetErrorString(e));
  }
  L->allocs.push_back(*p);
  (weight ? L->weight_bytes : L->ws_bytes) += (int64_t)bytes;
  return PI_OK;
}

static void free_all(pi_layer *L) {
  for (void *p : L->allocs) cudaFree(p);
  L->allocs.clear();
}

// ---------------------------------------------------------------------------
// type dispatch
// ---------------------------------------------------------------------------
template <int V>
using IC = std::integral_constant<int, V>;
template <typename T>
struct Tag {
  using type = T;
};

template <class F>
static pi_status dispatch_t(pi_dtype dt, F &&f) {
  if (dt == PI_DT_F16) return f(Tag<__half>{});
  if (dt == PI_DT_BF16) return f(Tag<__nv_bfloat16>{});
  return fail(PI_ERR_UNSUPPORTED, "dtype %d", (int)dt);
}

// ---------------------------------------------------------------------------
// ABI
// ---------------------------------------------------------------------------
extern "C" const char *pi_version(void) { return "libpi 0.1.0 sm_100a"; }
extern "C" const char *pi_last_error(void) { return g_err.c_str(); }

static bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }
static bool aligned2(const void *p) { return ((uintptr_t)p & 1u) == 0; }

extern "C" pi_status pi_layer_create(const pi_layer_desc *D, pi_stream_t stream, pi_layer **out) {
  g_err.clear();
  if (!out) return fail(PI_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!D) return fail(PI_ERR_INVALID_ARGUMENT, "desc is NULL");
  const int lid = D->layer_id;
  if (D->dtype != PI_DT_F16 && D->dtype != PI_DT_BF16)
    return fail(PI_ERR_UNSUPPORTED, "layer %d: dtype %d not supported", lid, (int)D->dtype);
  if (D->act != PI_ACT_RELU && D->act != PI_ACT_REGLU)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: act %d", lid, (int)D->act);
  if (D->pred_act != PI_PRED_RELU && D->pred_act != PI_PRED_LINEAR)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: pred_act %d", lid, (int)D->pred_act);
  if (D->d <= 0 || D->m_total <= 0 || D->rank <= 0 || D->m_local <= 0)
    return fail(PI_ERR_SHAPE, "layer %d: d=%d m_total=%d rank=%d m_local=%d must be > 0", lid, D->d,
                D->m_total, D->rank, D->m_local);
  if (D->d % 8 != 0) return fail(PI_ERR_ALIGNMENT, "layer %d: d=%d is not a multiple of 8", lid, D->d);
  if (D->rank % 8 != 0)
    return fail(PI_ERR_ALIGNMENT, "layer %d: rank=%d is not a multiple of 8", lid, D->rank);
  if (D->m_local > D->m_total)
    return fail(PI_ERR_SHAPE, "layer %d: m_local=%d > m_total=%d", lid, D->m_local, D->m_total);
  if (!D->neuron_ids && D->m_local != D->m_total)
    return fail(PI_ERR_SHAPE, "layer %d: neuron_ids NULL requires m_local == m_total (%d != %d)", lid,
                D->m_local, D->m_total);
  if (D->max_batch < 1 || D->max_batch > PI_MAX_BATCH)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: max_batch=%d not in 1..%d", lid, D->max_batch,
                PI_MAX_BATCH);
  if (D->ffn_format != PI_FFN_16 && D->ffn_format != PI_FFN_Q4)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: ffn_format %d", lid, (int)D->ffn_format);
  const bool q4 = D->ffn_format == PI_FFN_Q4;
  if (q4) {
    if (D->d % 32 != 0) return fail(PI_ERR_ALIGNMENT, "layer %d: PI_FFN_Q4 needs d %% 32 == 0 (d=%d)", lid, D->d);
    if (!D->w_up_scale || !D->w_down_scale || ((D->act == PI_ACT_REGLU) != (D->w_gate_scale != nullptr)))
      return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: PI_FFN_Q4 needs w_up_scale, w_down_scale (and w_gate_scale iff REGLU)",
                  lid);
    const void *sc[] = {D->w_up_scale, D->w_gate_scale, D->w_down_scale};
    for (const void *p : sc)
      if (p && !aligned2(p)) return fail(PI_ERR_ALIGNMENT, "layer %d: scale pointer %p not 2-B aligned", lid, p);
  } else if (D->w_up_scale || D->w_gate_scale || D->w_down_scale) {
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: *_scale pointers are only for PI_FFN_Q4", lid);
  }
  if (D->flags & ~(PI_FLAG_INPUT_RMSNORM | PI_FLAG_MULTI_KERNEL))
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: unknown flags 0x%x", lid, D->flags);
  if (D->max_batch > 8 && (q4 || D->d % 128 != 0))
    return fail(PI_ERR_UNSUPPORTED, "layer %d: max_batch=%d > 8 (the tensor-core batched path) needs 16-bit FFN "
                "weights and d %% 128 == 0 (d=%d)", lid, D->max_batch, D->d);
  if (std::isnan(D->logit_threshold))
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: logit_threshold is NaN", lid);
  if (!D->w_up || !D->w_down || !D->p_w1 || !D->p_w2)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: w_up, w_down, p_w1, p_w2 are required", lid);
  if ((D->act == PI_ACT_REGLU) != (D->w_gate != nullptr))
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: w_gate must be given iff act == REGLU", lid);
  const void *mats[] = {D->w_up, D->w_gate, D->w_down, D->p_w1, D->p_w2};
  for (const void *p : mats)
    if (p && !aligned16(p)) return fail(PI_ERR_ALIGNMENT, "layer %d: weight pointer %p not 16-B aligned", lid, p);
  const void *vecs[] = {D->b_up, D->b_down, D->p_b1, D->p_b2};
  for (const void *p : vecs)
    if (p && !aligned2(p)) return fail(PI_ERR_ALIGNMENT, "layer %d: bias pointer %p not 2-B aligned", lid, p);
  if (D->neuron_ids) {
    for (int k = 0; k < D->m_local; ++k) {
      const int v = D->neuron_ids[k];
      if (v < 0 || v >= D->m_total)
        return fail(PI_ERR_INDEX, "layer %d: neuron_ids[%d]=%d out of range [0,%d)", lid, k, v, D->m_total);
      if (k > 0 && v <= D->neuron_ids[k - 1])
        return fail(PI_ERR_INDEX, "layer %d: neuron_ids not strictly ascending at %d (%d after %d)", lid, k,
                    v, D->neuron_ids[k - 1]);
    }
  }
  int dev = 0;
  PI_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  PI_CUDA(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    return fail(PI_ERR_UNSUPPORTED, "layer %d: device %s is sm_%d%d; libpi is built for sm_100a", lid,
                prop.name, prop.major, prop.minor);

  pi_layer *L = new pi_layer();
  L->device = dev;
  L->num_sms = prop.multiProcessorCount;
  L->layer_id = lid;
  L->d = D->d;
  L->m_local = D->m_local;
  L->r = D->rank;
  L->words = (D->m_local + 31) / 32;
  L->max_batch = D->max_batch;
  L->dtype = D->dtype;
  L->ffn = D->ffn_format;
  L->rec_q4 = q4 ? (((int64_t)D->d / 2 + (int64_t)D->d / 16 + 15) / 16) * 16 : 0;
  L->act = D->act;
  L->pred_act = D->pred_act;
  L->flags = D->flags;
  L->threshold = D->logit_threshold;

  auto cleanup = [&](pi_status st) {
    free_all(L);
    delete L;
    return st;
  };
  const int d = L->d, ml = L->m_local, r = L->r, mt = D->m_total, MB = L->max_batch;
  const bool reglu = L->act == PI_ACT_REGLU;
  const size_t e = 2;
  pi_status st = PI_OK;
#define ALLOC(ptr, bytes, weight)                                          \
  do {                                                                     \
    st = dev_alloc(L, (void **)&(ptr), (size_t)(bytes), weight);           \
    if (st != PI_OK) return cleanup(st);                                   \
  } while (0)
  if (q4) {
    ALLOC(L->w_up, (size_t)ml * L->rec_q4 * (reglu ? 2 : 1), true);
    ALLOC(L->w_down, (size_t)ml * L->rec_q4, true);
  } else {
    ALLOC(L->w_up, (size_t)ml * d * e * (reglu ? 2 : 1), true);
    ALLOC(L->w_down, (size_t)ml * d * e, true);
  }
  if (D->b_up) ALLOC(L->b_up, (size_t)ml * e, true);
  if (D->b_down) ALLOC(L->b_down, (size_t)d * e, true);
  ALLOC(L->p_w1, (size_t)r * d * e, true);
  if (D->p_b1) ALLOC(L->p_b1, (size_t)r * e, true);
  // P2 in the fragment-major tile layout of the tensor-core GEMV (common.cuh): rows padded to whole
  // mask words, columns to 16
  ALLOC(L->p_w2, (size_t)L->words * 32 * ((r + 15) / 16 * 16) * e, true);
  if (D->p_b2) ALLOC(L->p_b2, (size_t)ml * e, true);

  // down-projection split: ~4 blocks per SM in total
  L->tiles = (d + 255) / 256;
  L->S = std::max(1, std::min(ml, (4 * L->num_sms + L->tiles - 1) / L->tiles));
  ALLOC(L->g, (size_t)MB * r * 4, false);
  ALLOC(L->scale, (size_t)MB * 4, false);
  ALLOC(L->h, (size_t)MB * ml * 4, false);
  ALLOC(L->partial, (size_t)L->S * MB * d * 4, false);
  if (MB >= 6 && !q4) ALLOC(L->upart, (size_t)((d + 255) / 256) * ml * 2 * std::min(MB, 8) * 4, false);
  ALLOC(L->tickets, (size_t)L->tiles * 4, false);
  ALLOC(L->mask, (size_t)MB * L->words * 4, false);
  ALLOC(L->ids, (size_t)ml * 4, false);
  ALLOC(L->n_active, 16, false);
  ALLOC(L->xbuf, (size_t)MB * d * 4, false);
  ALLOC(L->ybuf, (size_t)MB * d * 4, false);
  ALLOC(L->hx, (size_t)MB * d * 4, false);
  ALLOC(L->hy, (size_t)MB * d * 4, false);
  if (MB > 8) {
    const int bmax = MB <= 16 ? 16 : 32, N = 3 * bmax;
    L->S_tc = std::max(1, std::min(8, L->num_sms / std::max(1, d / 128)));
    ALLOC(L->x3, (size_t)d * N * 2, false);
    ALLOC(L->h3, (size_t)((ml + 63) / 64) * 64 * N * 2, false);
    ALLOC(L->partial_tc, (size_t)L->S_tc * bmax * d * 4, false);
    ALLOC(L->tickets_tc, (size_t)(d / 128) * 4, false);
  }
  // the fused kernel streams 16-bit rows or INT4 records (B = 1)
  if (!fused_alloc(L->fw, d, ml, r, MB, L->num_sms, reglu, [&](void **p, size_t bytes) {
        return dev_alloc(L, p, bytes, false) == PI_OK;
      }, q4 ? (int)L->rec_q4 : 0))
    return cleanup(fail(PI_ERR_OUT_OF_MEMORY, "layer %d: fused workspace", lid));
#undef ALLOC

  cudaStream_t s = (cudaStream_t)stream;
  L->hot_cap = D->hot_cap > 0 ? D->hot_cap : PI_DEFAULT_HOT_CAP;
  if (D->neuron_freq) {
    auto freq_of = [&](int k) { return D->neuron_freq[D->neuron_ids ? D->neuron_ids[k] : k]; };
    // speculative hot prefix: f >= spec_freq, hottest first (ties: ascending id), <= spec_cap
    std::vector<int32_t> spec;
    std::vector<uint8_t> is_spec(ml, 0);
    if (D->spec_freq > 0.f && D->spec_cap > 0 && L->fw.enabled) {
      for (int k = 0; k < ml; ++k)
        if (std::isfinite(freq_of(k)) && freq_of(k) >= D->spec_freq) spec.push_back(k);
      std::stable_sort(spec.begin(), spec.end(), [&](int a, int b) { return freq_of(a) > freq_of(b); });
      const int cap = std::min(D->spec_cap, kMaxSpecPerCta * L->num_sms);
      if ((int)spec.size() > cap) spec.resize(cap);
      for (int k : spec) is_spec[k] = 1;
    }
    if (!spec.empty()) {
      std::vector<uint32_t> words(L->words, 0u);
      for (int k : spec) words[k >> 5] |= 1u << (k & 31);
      st = dev_alloc(L, (void **)&L->spec_ids, spec.size() * 4, false);
      if (st != PI_OK) return cleanup(st);
      st = dev_alloc(L, (void **)&L->spec_words, (size_t)L->words * 4, false);
      if (st != PI_OK) return cleanup(st);
      if (cudaMemcpy(L->spec_ids, spec.data(), spec.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
          cudaMemcpy(L->spec_words, words.data(), words.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return cleanup(fail(PI_ERR_CUDA, "layer %d: speculative table copy", lid));
      L->n_spec = (int)spec.size();
    }
    // hot-neuron L2 prefetch list: f >= hot_freq, not speculative, hottest first
    std::vector<int32_t> hot;
    for (int k = 0; k < ml; ++k) {
      const float f = freq_of(k);
      if (!is_spec[k] && std::isfinite(f) && f >= D->hot_freq) hot.push_back(k);
    }
    std::stable_sort(hot.begin(), hot.end(), [&](int a, int b) { return freq_of(a) > freq_of(b); });
    if (!hot.empty()) {
      st = dev_alloc(L, (void **)&L->hot_ids, hot.size() * 4, false);
      if (st != PI_OK) return cleanup(st);
      if (cudaMemcpy(L->hot_ids, hot.data(), hot.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return cleanup(fail(PI_ERR_CUDA, "layer %d: hot table copy", lid));
      L->n_hot = (int)hot.size();
      std::vector<uint32_t> hw(L->words, 0u);
      for (int k = 0; k < std::min((int)hot.size(), L->hot_cap); ++k) hw[hot[k] >> 5] |= 1u << (hot[k] & 31);
      st = dev_alloc(L, (void **)&L->hot_words, hw.size() * 4, false);
      if (st != PI_OK) return cleanup(st);
      if (cudaMemcpy(L->hot_words, hw.data(), hw.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        return cleanup(fail(PI_ERR_CUDA, "layer %d: hot bitmap copy", lid));
    }
  }
  int32_t *d_nid = nullptr;
  if (D->neuron_ids) {
    if (cudaMalloc(&d_nid, (size_t)ml * 4) != cudaSuccess)
      return cleanup(fail(PI_ERR_OUT_OF_MEMORY, "layer %d: neuron table", lid));
    if (cudaMemcpyAsync(d_nid, D->neuron_ids, (size_t)ml * 4, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      cudaFree(d_nid);
      return cleanup(fail(PI_ERR_CUDA, "layer %d: neuron table copy", lid));
    }
  }
  cudaError_t ge = cudaSuccess;
  auto gather = [&](const void *src, void *dst, int cols, int64_t dst_stride, int dst_off) {
    const cudaError_t e = launch_gather_rows(src, d_nid, ml, cols, dst_stride, dst_off, dst, s);
    if (ge == cudaSuccess) ge = e;
  };
  if (q4) {
    auto pack = [&](const void *codes, const void *scales, void *dst, int64_t stride, int64_t off) {
      const cudaError_t e2 = launch_pack_q4(codes, scales, d_nid, ml, d, L->rec_q4, stride, off, dst, s);
      if (ge == cudaSuccess) ge = e2;
    };
    if (reglu) {
      pack(D->w_gate, D->w_gate_scale, L->w_up, 2 * L->rec_q4, 0);
      pack(D->w_up, D->w_up_scale, L->w_up, 2 * L->rec_q4, L->rec_q4);
    } else {
      pack(D->w_up, D->w_up_scale, L->w_up, L->rec_q4, 0);
    }
    pack(D->w_down, D->w_down_scale, L->w_down, L->rec_q4, 0);
  } else if (reglu) {
    gather(D->w_gate, L->w_up, d, 2 * (int64_t)d, 0);
    gather(D->w_up, L->w_up, d, 2 * (int64_t)d, d);
  } else {
    gather(D->w_up, L->w_up, d, d, 0);
  }
  {
    const cudaError_t e2 = launch_tile_p2(D->p_w2, d_nid, ml, r, L->p_w2, s);
    if (ge == cudaSuccess) ge = e2;
  }
  if (D->b_up) gather(D->b_up, L->b_up, 1, 1, 0);
  if (D->p_b2) gather(D->p_b2, L->p_b2, 1, 1, 0);
  if (!q4) {
    const cudaError_t e = launch_transpose_gather(D->w_down, d_nid, d, mt, ml, L->w_down, s);
    if (ge == cudaSuccess) ge = e;
  }
  cudaMemcpyAsync(L->p_w1, D->p_w1, (size_t)r * d * e, cudaMemcpyDeviceToDevice, s);
  if (D->p_b1) cudaMemcpyAsync(L->p_b1, D->p_b1, (size_t)r * e, cudaMemcpyDeviceToDevice, s);
  if (D->b_down) cudaMemcpyAsync(L->b_down, D->b_down, (size_t)d * e, cudaMemcpyDeviceToDevice, s);
  cudaMemsetAsync(L->tickets, 0, (size_t)L->tiles * 4, s);
  if (L->tickets_tc) cudaMemsetAsync(L->tickets_tc, 0, (size_t)(d / 128) * 4, s);
  cudaMemsetAsync(L->n_active, 0, 16, s);
  fused_init(L->fw, s);
  cudaError_t ce = cudaGetLastError();
  if (ce == cudaSuccess) ce = ge;
  if (d_nid) {
    // the table must outlive the async gathers (create is not on the hot path)
    cudaStreamSynchronize(s);
    cudaFree(d_nid);
  }
  if (ce != cudaSuccess) return cleanup(fail(PI_ERR_CUDA, "layer %d: repack: %s", lid, cudaGetErrorString(ce)));
  *out = L;
  return PI_OK;
}

extern "C" pi_status pi_layer_destroy(pi_layer *L) {
  g_err.clear();
  if (!L) return PI_OK;
  cudaDeviceSynchronize();
  free_all(L);
  delete L;
  return PI_OK;
}

static pi_status stack_dev(pi_layer *const *layers, int32_t n_layers, const float *x, int32_t B, float *y,
                           int32_t *n_out, cudaStream_t s);

static pi_status check_common(const pi_layer *L, int B);

// ---------------------------------------------------------------------------
// stacks: one persistent launch for L layers
// ---------------------------------------------------------------------------
struct pi_stack {
  std::vector<pi_layer *> layers;
  LayerW *lws = nullptr;  // device [L]
  bool fused = false;
  bool spec = false;      // some layer has a speculative hot prefix
};

extern "C" pi_status pi_stack_create(pi_layer *const *layers, int32_t n_layers, pi_stack **out) {
  g_err.clear();
  if (!out) return fail(PI_ERR_INVALID_ARGUMENT, "stack: out is NULL");
  *out = nullptr;
  if (!layers || n_layers < 1) return fail(PI_ERR_INVALID_ARGUMENT, "stack: NULL layers or n_layers < 1");
  const pi_layer *L0 = layers[0];
  if (!L0) return fail(PI_ERR_INVALID_ARGUMENT, "stack: layer 0 is NULL");
  for (int l = 0; l < n_layers; ++l) {
    const pi_layer *Ll = layers[l];
    if (!Ll) return fail(PI_ERR_INVALID_ARGUMENT, "stack: layer %d is NULL", l);
    if (Ll->d != L0->d || Ll->m_local != L0->m_local || Ll->r != L0->r || Ll->act != L0->act ||
        Ll->dtype != L0->dtype || Ll->pred_act != L0->pred_act || Ll->flags != L0->flags ||
        Ll->max_batch != L0->max_batch || Ll->device != L0->device)
      return fail(PI_ERR_SHAPE, "stack: layer %d (id %d) differs from layer 0 in shape/dtype/act/flags", l,
                  Ll->layer_id);
  }
  pi_stack *S = new pi_stack();
  S->layers.assign(layers, layers + n_layers);
  S->fused = !(L0->flags & PI_FLAG_MULTI_KERNEL) && L0->fw.enabled;
  std::vector<LayerW> h(n_layers);
  for (int l = 0; l < n_layers; ++l) {
    const pi_layer *Ll = layers[l];
    h[l].w_up = (const uint8_t *)Ll->w_up;
    h[l].w_down = (const uint8_t *)Ll->w_down;
    h[l].p_w1 = (const uint8_t *)Ll->p_w1;
    h[l].p_w2 = (const uint8_t *)Ll->p_w2;
    h[l].b_up = Ll->b_up;
    h[l].b_down = Ll->b_down;
    h[l].p_b1 = Ll->p_b1;
    h[l].p_b2 = Ll->p_b2;
    h[l].t = Ll->threshold;
    h[l].hot_ids = Ll->hot_ids;
    h[l].hot_words = Ll->hot_words;
    h[l].n_hot = std::min(Ll->n_hot, Ll->hot_cap);
    h[l].spec_ids = Ll->spec_ids;
    h[l].spec_words = Ll->spec_words;
    h[l].n_spec = Ll->n_spec;
    if (Ll->n_spec > 0) S->spec = true;
  }
  if (cudaMalloc(&S->lws, sizeof(LayerW) * n_layers) != cudaSuccess) {
    delete S;
    return fail(PI_ERR_OUT_OF_MEMORY, "stack: layer table");
  }
  if (cudaMemcpy(S->lws, h.data(), sizeof(LayerW) * n_layers, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(S->lws);
    delete S;
    return fail(PI_ERR_CUDA, "stack: layer table copy");
  }
  *out = S;
  return PI_OK;
}

extern "C" pi_status pi_stack_destroy(pi_stack *S) {
  g_err.clear();
  if (!S) return PI_OK;
  cudaDeviceSynchronize();
  cudaFree(S->lws);
  delete S;
  return PI_OK;
}

static pi_status stack_run_dev(pi_stack *S, const float *x, int B, float *y, int32_t *n_out, cudaStream_t s) {
  pi_layer *L0 = S->layers[0];
  const int n = (int)S->layers.size();
  if (S->fused && fused_supported(L0->fw, B)) {
    return dispatch_t(L0->dtype, [&](auto tt) {
      using T = typename decltype(tt)::type;
      FusedArgs a{};
      a.x = x; a.y = y; a.d = L0->d; a.m = L0->m_local; a.r = L0->r; a.words = L0->words; a.B = B;
      a.threshold = L0->threshold; a.rmsnorm = (L0->flags & PI_FLAG_INPUT_RMSNORM) != 0;
      a.pred_relu = L0->pred_act == PI_PRED_RELU; a.reglu = L0->act == PI_ACT_REGLU;
      a.n_out = n_out;
      a.hot_cap = L0->hot_cap;
      a.spec = S->spec;
      cudaError_t e = fused_launch_stack<T>(L0->fw, a, S->lws, n, s);
      if (e != cudaSuccess) return fail(PI_ERR_CUDA, "stack: fused launch: %s", cudaGetErrorString(e));
      return PI_OK;
    });
  }
  return stack_dev(S->layers.data(), n, x, B, y, n_out, s);
}

extern "C" pi_status pi_stack_run(pi_stack *S, const float *x, int32_t B, float *y, int32_t *n_active_out,
                                  pi_stream_t stream) {
  g_err.clear();
  if (!S) return fail(PI_ERR_INVALID_ARGUMENT, "stack handle is NULL");
  if (!x || !y) return fail(PI_ERR_INVALID_ARGUMENT, "stack: NULL x or y");
  PI_TRY(check_common(S->layers[0], B));
  if (!aligned16(x) || !aligned16(y)) return fail(PI_ERR_ALIGNMENT, "stack: x and y must be 16-B aligned");
  return stack_run_dev(S, x, B, y, n_active_out, (cudaStream_t)stream);
}

extern "C" pi_status pi_stack_run_host(pi_stack *S, const float *x_host, int32_t B, float *y_host,
                                       pi_stream_t stream) {
  g_err.clear();
  if (!S) return fail(PI_ERR_INVALID_ARGUMENT, "stack handle is NULL");
  if (!x_host || !y_host) return fail(PI_ERR_INVALID_ARGUMENT, "stack: NULL x_host or y_host");
  PI_TRY(check_common(S->layers[0], B));
  cudaStream_t s = (cudaStream_t)stream;
  pi_layer *L0 = S->layers[0];
  const size_t bytes = (size_t)B * L0->d * 4;
  PI_CUDA(cudaMemcpyAsync(L0->hx, x_host, bytes, cudaMemcpyHostToDevice, s));
  PI_TRY(stack_run_dev(S, L0->hx, B, L0->hy, nullptr, s));
  PI_CUDA(cudaMemcpyAsync(y_host, L0->hy, bytes, cudaMemcpyDeviceToHost, s));
  PI_CUDA(cudaStreamSynchronize(s));
  return PI_OK;
}

// ---------------------------------------------------------------------------
// groups: n_groups independent stacks in ONE persistent launch (SMs split into groups)
// ---------------------------------------------------------------------------
struct pi_group {
  std::vector<pi_layer *> layers;   // [n_groups * n_layers], group-major
  int n_groups = 0, n_layers = 0, group_ctas = 0;
  int defer = 0;                    // FusedParams.defer_ring from PI_GROUP_DEFER_*
  LayerW *lws = nullptr;            // device [n_groups * n_layers]
  FusedWork fw{};                   // geometry for P = group_ctas, buffers repeated per group
  std::vector<void *> allocs;
};

static void group_free(pi_group *G) {
  if (!G) return;
  for (void *p : G->allocs) cudaFree(p);
  if (G->lws) cudaFree(G->lws);
  delete G;
}

extern "C" pi_status pi_group_create(pi_layer *const *layers, int32_t n_groups, int32_t n_layers,
                                     int32_t group_ctas, uint32_t flags, pi_group **out) {
  g_err.clear();
  if (!out) return fail(PI_ERR_INVALID_ARGUMENT, "group: out is NULL");
  *out = nullptr;
  if (!layers || n_groups < 1 || n_layers < 1)
    return fail(PI_ERR_INVALID_ARGUMENT, "group: NULL layers, n_groups < 1 or n_layers < 1");
  const pi_layer *L0 = layers[0];
  if (!L0) return fail(PI_ERR_INVALID_ARGUMENT, "group: layer 0 is NULL");
  const int total = n_groups * n_layers;
  for (int i = 0; i < total; ++i) {
    const pi_layer *Ll = layers[i];
    if (!Ll) return fail(PI_ERR_INVALID_ARGUMENT, "group: layer %d is NULL", i);
    if (Ll->d != L0->d || Ll->m_local != L0->m_local || Ll->r != L0->r || Ll->act != L0->act ||
        Ll->dtype != L0->dtype || Ll->pred_act != L0->pred_act || Ll->flags != L0->flags ||
        Ll->device != L0->device || Ll->ffn != L0->ffn || Ll->n_spec != L0->n_spec)
      return fail(PI_ERR_SHAPE, "group: layer %d (id %d) differs from layer 0 in shape/dtype/act/flags/format", i,
                  Ll->layer_id);
  }
  if (L0->ffn != PI_FFN_16 || L0->n_spec > 0)
    return fail(PI_ERR_UNSUPPORTED, "group: grouped launches take 16-bit FFN rows without a speculative prefix");
  if (group_ctas < 1 || (int64_t)group_ctas * n_groups > L0->num_sms)
    return fail(PI_ERR_INVALID_ARGUMENT, "group: n_groups %d x group_ctas %d exceeds the %d SMs", n_groups,
                group_ctas, L0->num_sms);
  if (flags & ~(uint32_t)(PI_GROUP_DEFER_AFTER_REDUCTION | PI_GROUP_DEFER_AFTER_BARRIER) ||
      (flags & PI_GROUP_DEFER_AFTER_REDUCTION && flags & PI_GROUP_DEFER_AFTER_BARRIER))
    return fail(PI_ERR_INVALID_ARGUMENT, "group: unknown or conflicting flags 0x%x", flags);
  pi_group *G = new pi_group();
  G->defer = (flags & PI_GROUP_DEFER_AFTER_REDUCTION) ? 1 : (flags & PI_GROUP_DEFER_AFTER_BARRIER) ? 2 : 0;
  G->layers.assign(layers, layers + total);
  G->n_groups = n_groups;
  G->n_layers = n_layers;
  G->group_ctas = group_ctas;
  auto alloc = [&](void **p, size_t bytes) {
    if (cudaMalloc(p, bytes) != cudaSuccess) return false;
    G->allocs.push_back(*p);
    return true;
  };
  if (!fused_alloc(G->fw, L0->d, L0->m_local, L0->r, 1, group_ctas, L0->act == PI_ACT_REGLU, alloc, 0,
                   n_groups)) {
    group_free(G);
    return fail(PI_ERR_OUT_OF_MEMORY, "group: workspace");
  }
  if (!fused_supported(G->fw, 1) || !fused_group_supported(G->fw)) {
    group_free(G);
    return fail(PI_ERR_UNSUPPORTED, "group: shape d=%d m=%d r=%d has no grouped fused kernel for %d CTAs per group",
                L0->d, L0->m_local, L0->r, group_ctas);
  }
  std::vector<LayerW> h(total);
  for (int i = 0; i < total; ++i) {
    const pi_layer *Ll = layers[i];
    h[i] = LayerW{};
    h[i].w_up = (const uint8_t *)Ll->w_up;
    h[i].w_down = (const uint8_t *)Ll->w_down;
    h[i].p_w1 = (const uint8_t *)Ll->p_w1;
    h[i].p_w2 = (const uint8_t *)Ll->p_w2;
    h[i].b_up = Ll->b_up;
    h[i].b_down = Ll->b_down;
    h[i].p_b1 = Ll->p_b1;
    h[i].p_b2 = Ll->p_b2;
    h[i].t = Ll->threshold;
    h[i].hot_ids = Ll->hot_ids;
    h[i].hot_words = Ll->hot_words;
    h[i].n_hot = std::min(Ll->n_hot, Ll->hot_cap);
  }
  if (cudaMalloc(&G->lws, sizeof(LayerW) * total) != cudaSuccess ||
      cudaMemcpy(G->lws, h.data(), sizeof(LayerW) * total, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(G->fw.bar, 0, (size_t)n_groups * ((size_t)(1 + group_ctas) * 128 + 128)) != cudaSuccess) {
    group_free(G);
    return fail(PI_ERR_CUDA, "group: layer table / barrier init");
  }
  *out = G;
  return PI_OK;
}

extern "C" pi_status pi_group_destroy(pi_group *G) {
  g_err.clear();
  if (!G) return PI_OK;
  cudaDeviceSynchronize();
  group_free(G);
  return PI_OK;
}

extern "C" pi_status pi_group_run(pi_group *G, const float *x, int32_t B, float *y, int32_t *n_active_out,
                                  pi_stream_t stream) {
  g_err.clear();
  if (!G) return fail(PI_ERR_INVALID_ARGUMENT, "group handle is NULL");
  if (!x || !y) return fail(PI_ERR_INVALID_ARGUMENT, "group: NULL x or y");
  if (B != 1) return fail(PI_ERR_UNSUPPORTED, "group: grouped launches run B = 1 (got %d)", B);
  if (!aligned16(x) || !aligned16(y)) return fail(PI_ERR_ALIGNMENT, "group: x and y must be 16-B aligned");
  pi_layer *L0 = G->layers[0];
  return dispatch_t(L0->dtype, [&](auto tt) {
    using T = typename decltype(tt)::type;
    FusedArgs a{};
    a.x = x; a.y = y; a.d = L0->d; a.m = L0->m_local; a.r = L0->r; a.words = L0->words; a.B = B;
    a.threshold = L0->threshold; a.rmsnorm = (L0->flags & PI_FLAG_INPUT_RMSNORM) != 0;
    a.pred_relu = L0->pred_act == PI_PRED_RELU; a.reglu = L0->act == PI_ACT_REGLU;
    a.n_out = n_active_out;
    a.hot_cap = L0->hot_cap;
    FusedParams p = fused_params(G->fw, a);
    p.lws = G->lws;
    p.L = G->n_layers;
    p.mask = G->fw.mask;
    p.ids_out = nullptr;
    p.trace = L0->fw.trace;      // pi_layer_set_trace on layer 0: group 0's CTAs stamp their phases
    p.group_ctas = G->group_ctas;
    p.defer_ring = G->defer;
    cudaError_t e = fused_launch_p<T>(G->fw, p, a.reglu, B, (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(PI_ERR_CUDA, "group: fused launch: %s", cudaGetErrorString(e));
    return PI_OK;
  });
}

extern "C" pi_status pi_layer_set_trace(pi_layer *L, uint64_t *dev_buf) {
  g_err.clear();
  if (!L) return fail(PI_ERR_INVALID_ARGUMENT, "layer handle is NULL");
  L->fw.trace = reinterpret_cast<unsigned long long *>(dev_buf);
  return PI_OK;
}

extern "C" pi_status pi_layer_get_info(const pi_layer *L, pi_layer_info *info) {
  g_err.clear();
  if (!L || !info) return fail(PI_ERR_INVALID_ARGUMENT, "NULL argument");
  info->d = L->d;
  info->m_local = L->m_local;
  info->rank = L->r;
  info->max_batch = L->max_batch;
  info->mask_words = L->words;
  info->dtype = L->dtype;
  info->act = L->act;
  info->pred_act = L->pred_act;
  info->flags = L->flags;
  info->num_sms = L->num_sms;
  info->weight_bytes = L->weight_bytes;
  info->workspace_bytes = L->ws_bytes;
  info->ffn_format = L->ffn;
  info->n_spec = L->n_spec;
  info->launches_per_forward =
      (!(L->flags & PI_FLAG_MULTI_KERNEL) && fused_supported(L->fw, 1)) ? 1
                                                                        : 5 + ((L->flags & PI_FLAG_INPUT_RMSNORM) ? 1 : 0);
  return PI_OK;
}

static pi_status check_common(const pi_layer *L, int B) {
  if (!L) return fail(PI_ERR_INVALID_ARGUMENT, "layer handle is NULL");
  if (B < 1 || B > L->max_batch)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: batch %d not in 1..max_batch=%d", L->layer_id, B,
                L->max_batch);
  return PI_OK;
}

// scale pointer for the RMS flag (launches the scale kernel) or NULL
static const float *launch_scale(pi_layer *L, const float *x, int B, cudaStream_t s) {
  if (!(L->flags & PI_FLAG_INPUT_RMSNORM)) return nullptr;
  launch_rms_scale(x, B, L->d, L->scale, s);
  return L->scale;
}

static StepArgs step_args(const pi_layer *L) {
  StepArgs a{};
  a.p_w1 = L->p_w1; a.p_b1 = L->p_b1; a.p_w2 = L->p_w2; a.p_b2 = L->p_b2;
  a.w_up = L->w_up; a.b_up = L->b_up; a.w_down = L->w_down; a.b_down = L->b_down;
  a.g = L->g; a.h = L->h; a.partial = L->partial; a.tickets = L->tickets; a.upart = L->upart;
  a.d = L->d; a.m = L->m_local; a.r = L->r; a.kt = (L->r + 15) / 16; a.words = L->words; a.S = L->S; a.tiles = L->tiles;
  a.num_sms = L->num_sms; a.t = L->threshold;
  a.pred_relu = L->pred_act == PI_PRED_RELU; a.reglu = L->act == PI_ACT_REGLU;
  a.q4 = L->ffn == PI_FFN_Q4; a.rec_q4 = L->rec_q4;
  a.x3 = L->x3; a.h3 = L->h3; a.partial_tc = L->partial_tc; a.tickets_tc = L->tickets_tc; a.S_tc = L->S_tc;
  return a;
}

static pi_status cuda_status(cudaError_t e, const pi_layer *L, const char *what) {
  if (e == cudaSuccess) return PI_OK;
  return fail(PI_ERR_CUDA, "layer %d: %s launch: %s", L->layer_id, what, cudaGetErrorString(e));
}

static pi_status run_predict(pi_layer *L, const float *x, int B, const float *scale, uint32_t *mask,
                             float *logits, cudaStream_t s) {
  const StepArgs a = step_args(L);
  const cudaError_t e = L->dtype == PI_DT_F16 ? steps_predict<__half>(a, x, B, scale, mask, logits, s)
                                              : steps_predict<__nv_bfloat16>(a, x, B, scale, mask, logits, s);
  return cuda_status(e, L, "predict");
}

static pi_status run_ffn(pi_layer *L, const float *x, int B, const float *scale, const int32_t *ids,
                         const int32_t *n_active, const uint32_t *mask, float *y, cudaStream_t s) {
  const StepArgs a = step_args(L);
  const cudaError_t e = L->dtype == PI_DT_F16 ? steps_ffn<__half>(a, x, B, scale, ids, n_active, mask, y, s)
                                              : steps_ffn<__nv_bfloat16>(a, x, B, scale, ids, n_active, mask, y, s);
  return cuda_status(e, L, "sparse ffn");
}

extern "C" pi_status pi_predict(pi_layer *L, const float *x, int32_t B, uint32_t *mask, float *logits,
                                pi_stream_t stream) {
  g_err.clear();
  PI_TRY(check_common(L, B));
  if (!x || !mask) return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: x and mask are required", L->layer_id);
  if (!aligned16(x)) return fail(PI_ERR_ALIGNMENT, "layer %d: x not 16-B aligned", L->layer_id);
  cudaStream_t s = (cudaStream_t)stream;
  const float *scale = launch_scale(L, x, B, s);
  return run_predict(L, x, B, scale, mask, logits, s);
}

extern "C" pi_status pi_compact(pi_layer *L, const uint32_t *mask, int32_t B, int32_t *ids,
                                int32_t *n_active, pi_stream_t stream) {
  g_err.clear();
  PI_TRY(check_common(L, B));
  if (!mask || !ids || !n_active)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: mask, ids, n_active are required", L->layer_id);
  return cuda_status(launch_compact(mask, B, L->words, ids, n_active, (cudaStream_t)stream), L, "compact");
}

extern "C" pi_status pi_sparse_ffn(pi_layer *L, const float *x, int32_t B, const int32_t *ids,
                                   const int32_t *n_active, const uint32_t *mask, float *y,
                                   pi_stream_t stream) {
  g_err.clear();
  PI_TRY(check_common(L, B));
  if (!x || !ids || !n_active || !y)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: x, ids, n_active, y are required", L->layer_id);
  if (!mask && B != 1)
    return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: mask may be NULL only for B == 1 (B=%d)", L->layer_id, B);
  if (!aligned16(x) || !aligned16(y))
    return fail(PI_ERR_ALIGNMENT, "layer %d: x and y must be 16-B aligned", L->layer_id);
  cudaStream_t s = (cudaStream_t)stream;
  const float *scale = launch_scale(L, x, B, s);
  return run_ffn(L, x, B, scale, ids, n_active, mask, y, s);
}

static pi_status forward_dev(pi_layer *L, const float *x, int B, float *y, uint32_t *mask_out,
                             int32_t *ids_out, int32_t *n_out, cudaStream_t s) {
  if (!(L->flags & PI_FLAG_MULTI_KERNEL) && fused_supported(L->fw, B)) {
    return dispatch_t(L->dtype, [&](auto tt) {
      using T = typename decltype(tt)::type;
      FusedArgs a{};
      a.w_up = L->w_up; a.w_down = L->w_down; a.b_up = L->b_up; a.b_down = L->b_down;
      a.p_w1 = L->p_w1; a.p_b1 = L->p_b1; a.p_w2 = L->p_w2; a.p_b2 = L->p_b2;
      a.x = x; a.y = y; a.d = L->d; a.m = L->m_local; a.r = L->r; a.words = L->words; a.B = B;
      a.threshold = L->threshold; a.rmsnorm = (L->flags & PI_FLAG_INPUT_RMSNORM) != 0;
      a.pred_relu = L->pred_act == PI_PRED_RELU; a.reglu = L->act == PI_ACT_REGLU;
      a.mask_out = mask_out; a.ids_out = ids_out; a.n_out = n_out;
      a.hot_ids = L->hot_ids; a.hot_words = L->hot_words; a.n_hot = L->n_hot; a.hot_cap = L->hot_cap;
      cudaError_t e = fused_launch<T>(L->fw, a, L->num_sms, s);
      if (e != cudaSuccess) return fail(PI_ERR_CUDA, "layer %d: fused launch: %s", L->layer_id, cudaGetErrorString(e));
      return PI_OK;
    });
  }
  uint32_t *mask = mask_out ? mask_out : L->mask;
  int32_t *ids = ids_out ? ids_out : L->ids;
  int32_t *n = n_out ? n_out : L->n_active;
  const float *scale = launch_scale(L, x, B, s);
  PI_TRY(run_predict(L, x, B, scale, mask, nullptr, s));
  PI_TRY(cuda_status(launch_compact(mask, B, L->words, ids, n, s), L, "compact"));
  return run_ffn(L, x, B, scale, ids, n, mask, y, s);
}

extern "C" pi_status pi_layer_forward(pi_layer *L, const float *x, int32_t B, float *y, uint32_t *mask_out,
                                      int32_t *ids_out, int32_t *n_active_out, pi_stream_t stream) {
  g_err.clear();
  PI_TRY(check_common(L, B));
  if (!x || !y) return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: x and y are required", L->layer_id);
  if (!aligned16(x) || !aligned16(y))
    return fail(PI_ERR_ALIGNMENT, "layer %d: x and y must be 16-B aligned", L->layer_id);
  return forward_dev(L, x, B, y, mask_out, ids_out, n_active_out, (cudaStream_t)stream);
}

extern "C" pi_status pi_layer_forward_host(pi_layer *L, const float *x_host, int32_t B, float *y_host,
                                           pi_stream_t stream) {
  g_err.clear();
  PI_TRY(check_common(L, B));
  if (!x_host || !y_host) return fail(PI_ERR_INVALID_ARGUMENT, "layer %d: x_host and y_host are required", L->layer_id);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = (size_t)B * L->d * 4;
  PI_CUDA(cudaMemcpyAsync(L->hx, x_host, bytes, cudaMemcpyHostToDevice, s));
  PI_TRY(forward_dev(L, L->hx, B, L->hy, nullptr, nullptr, nullptr, s));
  PI_CUDA(cudaMemcpyAsync(y_host, L->hy, bytes, cudaMemcpyDeviceToHost, s));
  PI_CUDA(cudaStreamSynchronize(s));
  return PI_OK;
}

static pi_status stack_check(pi_layer *const *layers, int32_t n_layers, int32_t B) {
  if (!layers || n_layers < 1) return fail(PI_ERR_INVALID_ARGUMENT, "stack: NULL layers or n_layers < 1");
  for (int l = 0; l < n_layers; ++l) {
    PI_TRY(check_common(layers[l], B));
    if (layers[l]->d != layers[0]->d)
      return fail(PI_ERR_SHAPE, "stack: layer %d has d=%d, layer 0 has d=%d", layers[l]->layer_id,
                  layers[l]->d, layers[0]->d);
  }
  return PI_OK;
}

static pi_status stack_dev(pi_layer *const *layers, int32_t n_layers, const float *x, int32_t B, float *y,
                           int32_t *n_out, cudaStream_t s) {
  float *buf[2] = {layers[0]->xbuf, layers[0]->ybuf};
  const float *cur = x;
  for (int l = 0; l < n_layers; ++l) {
    float *dst = (l == n_layers - 1) ? y : buf[l & 1];
    if (cur == dst) dst = buf[(l + 1) & 1];
    PI_TRY(forward_dev(layers[l], cur, B, dst, nullptr, nullptr, n_out ? n_out + l : nullptr, s));
    cur = dst;
  }
  if (cur != y) PI_CUDA(cudaMemcpyAsync(y, cur, (size_t)B * layers[0]->d * 4, cudaMemcpyDeviceToDevice, s));
  return PI_OK;
}

extern "C" pi_status pi_stack_forward(pi_layer *const *layers, int32_t n_layers, const float *x, int32_t B,
                                      float *y, int32_t *n_active_out, pi_stream_t stream) {
  g_err.clear();
  if (!x || !y) return fail(PI_ERR_INVALID_ARGUMENT, "stack: NULL x or y");
  PI_TRY(stack_check(layers, n_layers, B));
  if (!aligned16(x) || !aligned16(y)) return fail(PI_ERR_ALIGNMENT, "stack: x and y must be 16-B aligned");
  return stack_dev(layers, n_layers, x, B, y, n_active_out, (cudaStream_t)stream);
}

extern "C" pi_status pi_stack_forward_host(pi_layer *const *layers, int32_t n_layers, const float *x_host,
                                           int32_t B, float *y_host, pi_stream_t stream) {
  g_err.clear();
  if (!x_host || !y_host) return fail(PI_ERR_INVALID_ARGUMENT, "stack: NULL x_host or y_host");
  PI_TRY(stack_check(layers, n_layers, B));
  cudaStream_t s = (cudaStream_t)stream;
  pi_layer *L0 = layers[0];
  const size_t bytes = (size_t)B * L0->d * 4;
  PI_CUDA(cudaMemcpyAsync(L0->hx, x_host, bytes, cudaMemcpyHostToDevice, s));
  PI_TRY(stack_dev(layers, n_layers, L0->hx, B, L0->hy, nullptr, s));
  PI_CUDA(cudaMemcpyAsync(y_host, L0->hy, bytes, cudaMemcpyDeviceToHost, s));
  PI_CUDA(cudaStreamSynchronize(s));
  return PI_OK;
}
