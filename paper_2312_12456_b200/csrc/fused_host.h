// fused_host.h -- host side of k_layer (fused.cuh): the whole hot path of one layer in ONE
// persistent, cooperative sm_100a kernel.
//
// One CTA per SM, 17 warps in three roles:
//   producer (warp 16) -- one elected lane streams every weight byte the CTA needs (its P1
//       rows, its block of P2 rows, then the up(/gate) and down rows of its share of the
//       active neurons) with 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP) into an
//       NS-stage shared-memory ring guarded by full/empty mbarriers;
//   up group (warps 0..7, 256 threads) -- owns x in registers (fixed 16-byte column chunks
//       of d per thread); computes the P1 row dots and, per ring stage, the up (and gate)
//       dots of the stage's neurons: per-warp transpose reductions, one 256-thread named
//       barrier per stage, then h = act(.) is handed to the down group through shared
//       memory and an "h ready" mbarrier;
//   down group (warps 8..15, 256 threads) -- computes the P2 GEMV + threshold + ballot
//       (one warp per ring stage of mask words, transpose-reduced), then, per FFN stage,
//       accumulates h * down-row into its register-resident partial y.
// The two groups are decoupled by the ring: the up group runs ahead of the down group.
//
//   phase 1  g = act_p(s * P1 x + b1)                rows of P1 dealt round-robin to CTAs
//   -------- grid barrier 1 (g visible)
//   phase 2  z = P2 g + b2 ; bit = z > t ; ballot     contiguous block of mask words per CTA
//            union words + per-CTA popcount
//   -------- grid barrier 2 (mask, union, counts visible)
//   phase 3  every CTA prefix-sums the counts, takes compacted positions
//            [c n / P, (c+1) n / P) -- equal work, since every compacted neuron costs the
//            same -- extracts its ids from the union words, and streams up + down rows:
//            h = act(s * W_up[i] x + b_up[i]) (per-token bit), y_part += h * Wd_T[i]
//   -------- grid barrier 3 (per-CTA partials visible)
//   phase 4  CTA c reduces its column slice over the P partials in fixed order, + b_down
//
// The producer runs ahead across barriers 1 and 2 for P2 rows (data-independent), so those
// bytes stream in while the grid synchronises.  All reductions have a fixed order: the
// result is bitwise reproducible run to run; there are no float atomics.
#pragma once

#include <algorithm>

#include "common.cuh"

namespace pi {

constexpr int kGroupWarps = 8;                        // warps per group (up / down)
constexpr int kGroup = kGroupWarps * 32;              // 256 threads per group
constexpr int kConsumerWarps = 2 * kGroupWarps;       // 16
constexpr int kConsumers = kConsumerWarps * 32;       // 512
constexpr int kFusedThreads = kConsumers + 32;        // + producer warp
constexpr int kFusedMaxB = 2;
constexpr int kMaxCH = 8;        // 16-byte chunks of d per group thread (d <= 16384)
constexpr int kMaxWordsP2 = 16;  // P2 mask words per stage (4 jobs per word: 2 row tiles x 2 K halves)
constexpr int kRedStride = 32;   // floats per warp in the up-group reduction buffer
constexpr int kMaxStages = 16;   // ring stages (s_slot_pos)
constexpr int kMaxSpecPerCta = 32;   // speculative hot-prefix neurons per CTA (static shared tables)
constexpr int kMaxCorrPerCta = 32;   // corrections per CTA and layer (more: the rest run unspeculated)
constexpr int kMaxP1PerCta = 64;     // predictor hidden rows per CTA (s_b1)

struct FusedWork {
  bool enabled = false;
  int P = 0, NS = 0, stage_bytes = 0, words_p2 = 0, idcap = 0, wcap = 0, smem = 0, part_off = 0, pcap = 0, kt = 0;
  int d = 0, m = 0, r = 0;
  bool reglu = false;
  unsigned long long *bar = nullptr;  // grid barrier counter (monotonic)
  float *g = nullptr;                 // [maxB, r]
  float *ypart = nullptr;             // [P, maxB, d]
  int rec_q4 = 0;                     // INT4 FFN records: bytes per neuron and matrix (0 = 16-bit rows)
  int *counts = nullptr;              // [P]
  int *counts_full = nullptr;         // [P]
  uint32_t *mask = nullptr;           // [maxB, words]
  uint32_t *uni = nullptr;            // [words]
  float *xbuf = nullptr;              // [maxB, d] inter-layer activations (stack launch)
  unsigned long long *trace = nullptr;  // optional phase trace (pi_layer_set_trace)
  int groups = 1;                     // grouped workspace (pi_group): buffers repeated per group
};

struct FusedArgs {
  const void *w_up, *w_down, *b_up, *b_down, *p_w1, *p_b1, *p_w2, *p_b2;
  const float *x;
  float *y;
  int d, m, r, words, B;
  float threshold;
  bool rmsnorm, pred_relu, reglu;
  uint32_t *mask_out;
  int32_t *ids_out, *n_out;
  const int32_t *hot_ids;
  const uint32_t *hot_words;
  int n_hot, hot_cap;
  bool spec;   // stack launch whose layers carry speculative tables
};

struct LayerW {  // one layer's library-owned weights (device pointers)
  const uint8_t *w_up, *w_down, *p_w1, *p_w2;
  const void *b_up, *b_down, *p_b1, *p_b2;
  const int32_t *hot_ids;   // local ids of the hot neurons (L2-prefetched each step), or NULL
  const uint32_t *hot_words;  // [words] bitmap of the prefetched hot neurons (FFN order: hot first), or NULL
  int n_hot;
  float t;
  const int32_t *spec_ids;      // speculative hot prefix (hottest first), or NULL
  const uint32_t *spec_words;   // [words] bitmap of the speculative neurons
  int n_spec;
};

struct FusedParams {
  LayerW lw0;                 // the layer of a single-layer launch
  const LayerW *lws;          // device array of L layers (stack launch) or NULL (use lw0)
  int L;
  const float *x;             // layer-0 input [B, d]
  float *y;                   // last-layer output [B, d]
  float *xbuf;                // inter-layer activations [B, d] (stack launch)
  int d, m, r, words, B;
  int rmsnorm, pred_relu;
  uint32_t *mask, *uni;
  int32_t *ids_out, *n_out;   // n_out: [L] union counts
  float *g, *ypart;
  int *counts;
  int *counts_full;           // [P] per-CTA union counts incl. the speculative neurons
  unsigned long long *bar;
  int spec;                   // speculative hot prefix on (stack launches only)
  int NS, stage_bytes, G, rows_p1, words_p2, idcap, wcap, part_off, pcap;
  int kt;                     // 16-column K tiles of the fragment-major P2 (ceil(r / 16))
  int rec_q4;                 // INT4 FFN records (bytes per neuron and matrix); 0 = 16-bit rows
  unsigned long long *trace;  // [P][256] timestamps (globaltimer ns) of layer 0, or NULL
  int hot_cap;                // at most this many hot neurons are L2-prefetched per layer
  int defer_ring;             // 0: the producer runs ahead into the next layer; 1 / 2: it waits for the
                              // previous layer's reduction / last grid barrier (pi_group_create flags)
  int group_ctas;             // > 0: grouped launch (pi_group_run) -- the grid is n_groups independent
                              // problems of group_ctas CTAs each; group k uses lws + k L, x/y + k B d and
                              // the k-th slice of every workspace buffer (strides: fused.cuh group_view)
};

// Everything below is host code (kernel launch parameters, workspace sizing, dispatch); the
// kernel itself is in fused.cuh, compiled once per (weight type, batch) instantiation unit.
// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
inline int fused_ch(int d) { return (d / 8 + kGroup - 1) / kGroup; }
// phase-4 partial-sum buffer (floats): [SPL][columns x B / 4][4] with SPL <= max(ceil(P / 8), 512 / items)
__host__ __device__ constexpr int fused_spart(int P, int pcap, int B) {
  return ((P + 7) / 8) * pcap * B > 4 * kConsumers ? ((P + 7) / 8) * pcap * B : 4 * kConsumers;
}

template <class Alloc>
inline bool fused_alloc(FusedWork &w, int d, int m, int r, int maxB, int num_sms, bool reglu, Alloc &&alloc,
                        int rec_q4 = 0, int groups = 1) {
  w = FusedWork{};
  w.groups = groups;
  w.rec_q4 = rec_q4;
  w.d = d;
  w.m = m;
  w.r = r;
  w.reglu = reglu;
  const int ch = fused_ch(d);
  if (ch > kMaxCH || d < 8 || r > kMaxP1PerCta * num_sms || num_sms > 256)
    return true;  // unsupported shape: stays disabled (per-step kernels)
  w.P = num_sms;
  w.kt = (r + 15) / 16;
  const size_t p2_word = (size_t)32 * w.kt * 16 * 2;   // one 32-row word of the tiled P2
  // stage: >= one P2 word, >= 32 KB, and a whole number NA of neurons (gate|up + down; NA a power of
  // two <= 8, as many as ~40 KB hold) so no neuron slot of the instantiated kernel idles
  const size_t nb = rec_q4 ? (size_t)rec_q4 * (reglu ? 3 : 2) : (size_t)d * (reglu ? 6 : 4);
  size_t na = 1;
  while (na < 8 && 2 * na * nb <= (size_t)(rec_q4 ? 48 : 40) * 1024) na *= 2;
  size_t sb = std::max<size_t>({(size_t)32 * 1024, na * nb, p2_word});
  sb = (sb + 127) / 128 * 128;
  // compaction stages the union words, the per-token words, the hot bitmap and the P counts in one ring slot
  if ((size_t)((m + 31) / 32) * (2 + kFusedMaxB) * 4 + (size_t)2 * num_sms * 4 > sb) return true;
  w.stage_bytes = (int)sb;
  w.words_p2 = std::min<int>(kMaxWordsP2, (int)(sb / p2_word));
  w.idcap = (m + w.P - 1) / w.P + 2;
  const int words_all = (m + 31) / 32;
  w.wcap = (words_all + w.P - 1) / w.P + 1;
  w.pcap = ((d / 8 + w.P - 1) / w.P + 1) * 8;   // phase-4 columns per CTA (8-column units), upper bound
  const int mb = std::max(1, std::min(maxB, kFusedMaxB));   // the kernel's B <= max_batch
  const int NT = (3 * mb + 7) / 8;
  // everything but the ring: mbarriers, reduction buffers, h, logits, b2, b_up/ids/bits, phase-4
  // partials, g staging and its B fragments; the ring gets the rest (<= 200 KB)
  // B = 2 kernels keep x in shared memory ([B][d] fp32, fused.cuh s_x) instead of registers
  const size_t xs_bytes = mb >= 2 ? (size_t)mb * d * 4 : 0;
  auto extras = [&](int ns) {
    return (size_t)(3 * ns + 2) * 8 + (size_t)2 * kGroupWarps * kRedStride * 4 + (size_t)ns * 8 * mb * 4 +
           (size_t)(2 * mb + 1) * w.wcap * 32 * 4 + (size_t)w.idcap * 9 + 16 + (size_t)fused_spart(w.P, w.pcap, mb) * 4 +
           (size_t)mb * w.kt * 16 * 4 + (size_t)w.kt * NT * 32 * 8 + xs_bytes + 64;
  };
  const size_t cap = 227 * 1024 - 2560;   // static shared memory (speculative tables, barriers) and slack
  w.NS = (int)std::min<size_t>({200 * 1024 / sb, cap / sb, (size_t)kMaxStages});
  if ((size_t)w.kt * 12 * mb > (size_t)3 * kConsumers) return true;   // p2_phase: <= 3 entries per thread
  while (w.NS >= 2 && (size_t)w.NS * sb + extras(w.NS) > cap) --w.NS;
  if (w.NS < 2) return true;
  const size_t pre = (size_t)(3 * w.NS + 2) * 8 + (size_t)2 * kGroupWarps * kRedStride * 4 +
                     (size_t)w.NS * 8 * mb * 4 + (size_t)(2 * mb + 1) * w.wcap * 32 * 4 + (size_t)w.idcap * 9;
  w.part_off = (int)(((size_t)w.NS * sb + pre + 15) / 16 * 16);
  w.smem = w.part_off + fused_spart(w.P, w.pcap, mb) * 4 + mb * w.kt * 16 * 4 + w.kt * NT * 32 * 8 + (int)xs_bytes + 64;
  const int words = (m + 31) / 32;
  // a grouped workspace repeats every buffer per group with the strides of fused.cuh group_view
  const size_t G = (size_t)groups;
  const int gb = groups > 1 ? kFusedMaxB : maxB;
  if (!alloc((void **)&w.bar, G * ((size_t)(1 + num_sms) * 128 + 128))) return false;
  if (!alloc((void **)&w.g, G * (size_t)gb * r * 4)) return false;
  if (!alloc((void **)&w.ypart, G * (size_t)w.P * std::min(gb, kFusedMaxB) * d * 4)) return false;
  if (!alloc((void **)&w.counts, G * (size_t)w.P * 4)) return false;
  if (!alloc((void **)&w.counts_full, G * (size_t)w.P * 4)) return false;
  if (!alloc((void **)&w.mask, G * (size_t)gb * words * 4)) return false;
  if (!alloc((void **)&w.uni, G * (size_t)words * 4)) return false;
  if (!alloc((void **)&w.xbuf, G * (size_t)std::min(gb, kFusedMaxB) * d * 4)) return false;
  if (w.smem > 227 * 1024) return true;
  w.enabled = true;
  return true;
}

inline void fused_init(FusedWork &w, cudaStream_t s) {
  if (w.enabled) cudaMemsetAsync(w.bar, 0, (size_t)w.groups * ((size_t)(1 + w.P) * 128 + 128), s);
}

// max P1 rows per stage of the kernel (its unrolled row loop): ~one 32 KB stage of d-rows
__host__ __device__ constexpr int fused_rpm(int ch) { return ch >= 8 ? 1 : (8 / ch > 8 ? 8 : 8 / ch); }

// neurons per stage (NA template bound and runtime G) and P1 rows per stage
inline void fused_geometry(const FusedWork &w, int d, bool reglu, int *NA, int *G, int *RP1) {
  const size_t nb = w.rec_q4 ? (size_t)w.rec_q4 * (reglu ? 3 : 2) : (size_t)d * 2 * (reglu ? 3 : 2);
  const int g = (int)std::min<size_t>(8, w.stage_bytes / nb);
  // neurons per stage: the largest power of two <= 8 the stage holds (the kernel's unrolled
  // neuron loop is exactly NA long, so no slot computes on padding)
  *NA = g >= 8 ? 8 : g >= 4 ? 4 : g >= 2 ? 2 : 1;
  *G = *NA;
  const int rp = (int)(w.stage_bytes / ((size_t)d * 2));
  *RP1 = std::max(1, std::min(fused_rpm(fused_ch(d)), rp));
}

inline bool fused_supported(const FusedWork &w, int B = 1) {
  if (!w.enabled || B < 1 || B > kFusedMaxB) return false;
  if (w.rec_q4 && B != 1) return false;   // INT4 rows: the fused kernel is instantiated for B = 1
  const int ch = fused_ch(w.d);
  if (ch * 8 * B > 64) return false;  // register-resident x / y per group thread
  int NA, G, RP1;
  fused_geometry(w, w.d, w.reglu, &NA, &G, &RP1);
  // the instantiated (CH, NA) combinations (fused_launch_tbr)
  if (w.rec_q4)   // INT4 records: fused.cuh fused_launch_t's Q4 list
    return (ch <= 2 && NA >= 4) || ((ch == 3 || ch == 4) && NA == 4) || (ch >= 5 && NA == 2);
  if (ch <= 2) return true;
  if (NA == 1) return ch <= 4 || (B == 1 && ch <= kMaxCH);
  return false;
}

// the grouped kernel (fused.cuh fused_launch_t) is instantiated for B = 1, d <= 8192 (CH <= 4), NA 1 or 8
inline bool fused_group_supported(const FusedWork &w) {
  if (!w.enabled || w.rec_q4) return false;
  int NA, G, RP1;
  fused_geometry(w, w.d, w.reglu, &NA, &G, &RP1);
  const int ch = fused_ch(w.d);
  return ch <= 2 || (ch <= 4 && NA == 1);
}

// One instantiation unit per (weight type, batch, activation): fused_inst_<T>_b<B>_<act>.cu
// defines it from fused.cuh.
template <typename T, int B, bool REGLU>
cudaError_t fused_launch_tbr(const FusedWork &w, const FusedParams &p, int CH, int NA, cudaStream_t s);
template <typename T, int B>
inline cudaError_t fused_launch_tb(const FusedWork &w, const FusedParams &p, bool reglu, int CH, int NA,
                                   cudaStream_t s) {
  return reglu ? fused_launch_tbr<T, B, true>(w, p, CH, NA, s) : fused_launch_tbr<T, B, false>(w, p, CH, NA, s);
}

// Parameters shared by the single-layer and the stack launch.
inline FusedParams fused_params(const FusedWork &w, const FusedArgs &a) {
  FusedParams p{};
  p.lw0.w_up = (const uint8_t *)a.w_up;
  p.lw0.w_down = (const uint8_t *)a.w_down;
  p.lw0.p_w1 = (const uint8_t *)a.p_w1;
  p.lw0.p_w2 = (const uint8_t *)a.p_w2;
  p.lw0.b_up = a.b_up;
  p.lw0.b_down = a.b_down;
  p.lw0.p_b1 = a.p_b1;
  p.lw0.p_b2 = a.p_b2;
  p.lw0.t = a.threshold;
  p.lw0.hot_ids = a.hot_ids;
  p.lw0.hot_words = a.hot_words;
  p.lw0.n_hot = a.n_hot;
  p.lws = nullptr;
  p.L = 1;
  p.x = a.x;
  p.y = a.y;
  p.xbuf = w.xbuf;
  p.d = a.d;
  p.m = a.m;
  p.r = a.r;
  p.words = a.words;
  p.B = a.B;
  p.rmsnorm = a.rmsnorm;
  p.pred_relu = a.pred_relu;
  p.mask = a.mask_out ? a.mask_out : w.mask;
  p.uni = w.uni;
  p.ids_out = a.ids_out;
  p.n_out = a.n_out;
  p.g = w.g;
  p.ypart = w.ypart;
  p.counts = w.counts;
  p.counts_full = w.counts_full;
  p.bar = w.bar;
  p.NS = w.NS;
  p.stage_bytes = w.stage_bytes;
  p.words_p2 = w.words_p2;
  p.idcap = w.idcap;
  p.wcap = w.wcap;
  p.part_off = w.part_off;
  p.pcap = w.pcap;
  p.kt = w.kt;
  p.rec_q4 = w.rec_q4;
  p.trace = w.trace;
  p.hot_cap = a.hot_cap;
  return p;
}

template <typename T>
inline cudaError_t fused_launch_p(FusedWork &w, FusedParams p, bool reglu, int B, cudaStream_t s) {
  int NA, G, RP1;
  fused_geometry(w, p.d, reglu, &NA, &G, &RP1);
  p.G = G;
  p.rows_p1 = RP1;
  const int CH = fused_ch(p.d);
  if (B == 1) return fused_launch_tb<T, 1>(w, p, reglu, CH, NA, s);
  if (B == 2) return fused_launch_tb<T, 2>(w, p, reglu, CH, NA, s);
  return cudaErrorNotSupported;
}

// one layer
template <typename T>
inline cudaError_t fused_launch(FusedWork &w, const FusedArgs &a, int /*num_sms*/, cudaStream_t s) {
  return fused_launch_p<T>(w, fused_params(w, a), a.reglu, a.B, s);
}

// L chained layers in one launch: a describes layer 0 (shapes, x, y); lws is a device array of
// the L layers' weights; n_out (optional) receives the L union counts.
template <typename T>
inline cudaError_t fused_launch_stack(FusedWork &w, const FusedArgs &a, const LayerW *lws, int L,
                                      cudaStream_t s) {
  FusedParams p = fused_params(w, a);
  p.lws = lws;
  p.L = L;
  p.mask = w.mask;
  p.ids_out = nullptr;
  p.spec = a.spec ? 1 : 0;   // the SPEC kernel variant; layers with n_spec == 0 run unspeculated in it
  return fused_launch_p<T>(w, p, a.reglu, a.B, s);
}

}  // namespace pi
