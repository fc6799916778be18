// verify.cu — dsde_verify: the fused speculative-verification pass (§8(a) a1-a4).
//
// Pipeline (all on the caller's stream, no host synchronisation; 3 launches):
//   1. k_stream_tma   persistent CTAs, TMA-bulk ring: one streaming read of every
//                     (draft position row, vocab chunk) of the target and draft
//                     logits; chunk max/argmax, then S = sum e_v, A = sum e_v w_v,
//                     D = sum e_v g(w_v) about the chunk reference (a1).
//   2. k_finalize     one warp per sequence, one lane per position: fp64 merge of
//                     the chunk partials about the row reference, KL, log p/q, the
//                     Philox accept test, the first rejection a_i, token layout (a2-a3).
//   3. k_sample       per (sequence, chunk): draw-weight mass of the residual
//                     max(0, p - q) (row a_i) or of p (bonus row k_i); the last CTA
//                     of each sequence selects the smallest token with C_v > u R (a4, D7).
//
// Numerics: with e_v = exp(t_v - M), w_v = (t_v - d_v) - C, C = t - d at
// the argmax of t, and g(w) = exp(-w) - 1 + w >= 0:
//   KL(p||q) = D/S + (log1p(y) - y),  y = (D - A)/S = E_p[exp(-w)] - 1,
//   log p(x)/q(x) = (t_x - d_x) - C + log1p(y),
//   q_v / p_v = exp(-(w_v + log1p(y))).
// D sums non-negative terms, so the small-KL regime has no cancellation (the naive
// E_p[t - d] - LSE_t + LSE_d form loses ~1e-3 relative at KL ~ 1e-3).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cuda_bf16.h>

#include "common.cuh"
#include "state.cuh"

namespace dsde {

constexpr int kThreads = 256;

template <typename T>
struct Traits;
template <>
struct Traits<uint16_t> {      // bf16 bit patterns
  static constexpr int VEC = 8;  // elements per 16-byte vector
  static constexpr int NV = 4;   // vectors per thread per row
};
template <>
struct Traits<float> {
  static constexpr int VEC = 4;
  static constexpr int NV = 4;
};
template <typename T>
__host__ __device__ constexpr int chunk_elems() {
  return kThreads * Traits<T>::VEC * Traits<T>::NV;
}

struct ChunkPartial {  // 48 bytes
  double S, A, D;      // about (M, C) of this chunk
  float M;             // chunk max of t
  float C;             // t - d at the chunk argmax (fp32, as used for w)
  int idx;             // chunk argmax (smallest index among ties)
  int flags;           // DSDE_FLAG_OVERFLOW
  float maxd;          // max of d over the chunk (overflow-safe reference bound)
  int pad;
};
static_assert(sizeof(ChunkPartial) == 48, "ChunkPartial layout");

enum { MODE_NONE = 0, MODE_RESIDUAL = 1, MODE_BONUS = 2, MODE_ERROR = 3 };

struct SeqRec {  // 64 bytes
  int mode;
  int slot;          // output slot of the drawn token, cu_sl[i] + i + a_i
  long long trow;    // target row to draw from
  long long drow;    // draft row (residual only)
  float M;           // reference max of t (residual)
  int pad0;
  double C;          // reference t - d (residual)
  double lam;        // log1p(y) = log(sum_v p_v exp(-w_v)) (residual)
  double u;          // u_smp of the slot
  double pad1;
};
static_assert(sizeof(SeqRec) == 64, "SeqRec layout");

struct VerifyWs {
  ChunkPartial* part;  // [(total + B) * nchunks]
  SeqRec* rec;         // [B]
  double* mass;        // [B * nchunks * 8] draw-weight mass per warp sub-chunk
  float* cmax;         // [B * nchunks * 8] reference of each sub-chunk mass (bonus)
  int* counter;        // [3 * B] per-sequence counters / flags (zeroed per call)
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

inline int n_chunks(int V, dsde_dtype dt) {
  const int ch = dt == DSDE_BF16 ? chunk_elems<uint16_t>() : chunk_elems<float>();
  return (V + ch - 1) / ch;
}

inline size_t ws_layout(int B, int total, int V, dsde_dtype dt, VerifyWs* ws, char* base) {
  const int nc = n_chunks(V, dt);
  size_t off = 0;
  const size_t p_bytes = align256(sizeof(ChunkPartial) * (size_t)(total + B) * nc);
  const size_t r_bytes = align256(sizeof(SeqRec) * (size_t)B);
  const size_t m_bytes = align256(sizeof(double) * (size_t)B * nc * 8);  // per warp sub-chunk
  const size_t x_bytes = align256(sizeof(float) * (size_t)B * nc * 8);
  const size_t c_bytes = align256(sizeof(int) * ((size_t)B * 5 + 8));  // counters + event queue
  if (ws) {
    ws->part = reinterpret_cast<ChunkPartial*>(base + off);
    ws->rec = reinterpret_cast<SeqRec*>(base + off + p_bytes);
    ws->mass = reinterpret_cast<double*>(base + off + p_bytes + r_bytes);
    ws->cmax = reinterpret_cast<float*>(base + off + p_bytes + r_bytes + m_bytes);
    ws->counter = reinterpret_cast<int*>(base + off + p_bytes + r_bytes + m_bytes + x_bytes);
  }
  return p_bytes + r_bytes + m_bytes + x_bytes + c_bytes;
}

template <typename T>
__device__ __forceinline__ float load_logit_smem(const T* p);
template <>
__device__ __forceinline__ float load_logit_smem<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float load_logit_smem<uint16_t>(const uint16_t* p) {
  return bf16_bits_to_float(*p);
}

// max that propagates NaN (a NaN logit must reach the non-finite check)
__device__ __forceinline__ float max_nan(float a, float b) { return (b > a || b != b) ? b : a; }

__device__ __forceinline__ void arg_better(float& m, int& mi, float& md, float m2, int i2, float d2) {
  if (m2 > m || (m2 == m && i2 < mi)) {
    m = m2;
    mi = i2;
    md = d2;
  }
}

// w = (t - d) - C. For bf16 inputs t - d is exact in fp32 (8-bit significands,
// exponent gap <= 16 in practice); for fp32 inputs the difference is carried as
// an unevaluated sum (TwoDiff, Knuth) so w keeps full fp32 accuracy.
template <typename T>
__device__ __forceinline__ float diff_ref(float t, float d, float C);
template <>
__device__ __forceinline__ float diff_ref<uint16_t>(float t, float d, float C) {
  return (t - d) - C;
}
template <>
__device__ __forceinline__ float diff_ref<float>(float t, float d, float C) {
  const float hi = __fsub_rn(t, d);
  const float bb = __fsub_rn(hi, t);
  const float lo = __fadd_rn(__fsub_rn(t, __fsub_rn(hi, bb)), __fsub_rn(-d, bb));
  return __fadd_rn(__fsub_rn(hi, C), lo);
}

// ---------------------------------------------------------------------------
// mbarrier / TMA bulk-copy primitives (PTX), packed element helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// Blocking wait on an mbarrier phase (try_wait blocks in hardware for a
// system-defined time before returning false; the loop re-probes).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

struct StreamTmaArgs {
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const int32_t* cu_sl;
  int B, V, nchunks, total;
  ChunkPartial* part;
};

template <typename T>
__host__ __device__ constexpr int stage_row_bytes() {
  return chunk_elems<T>() * (int)sizeof(T);
}

template <typename T>
__device__ __forceinline__ void unpack16(uint4 raw, float* x);
template <>
__device__ __forceinline__ void unpack16<uint16_t>(uint4 raw, float* x) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    x[2 * h] = bf16_lo(w[h]);
    x[2 * h + 1] = bf16_hi(w[h]);
  }
}
template <>
__device__ __forceinline__ void unpack16<float>(uint4 raw, float* x) {
  x[0] = __uint_as_float(raw.x);
  x[1] = __uint_as_float(raw.y);
  x[2] = __uint_as_float(raw.z);
  x[3] = __uint_as_float(raw.w);
}

template <typename T>
__device__ __forceinline__ T pad_bits();
template <>
__device__ __forceinline__ uint16_t pad_bits<uint16_t>() { return (uint16_t)0xF14Au; }  // bf16 ~ -1e30
template <>
__device__ __forceinline__ float pad_bits<float>() { return -1e30f; }

// Elements h, h+1 (h even) of a lane's 4 x 16-byte vectors as an fp32 pair.
template <typename T>
__device__ __forceinline__ float2 pair_of(const uint4 (&r)[Traits<T>::NV], int h);
template <>
__device__ __forceinline__ float2 pair_of<uint16_t>(const uint4 (&r)[4], int h) {
  const uint4 x = r[h >> 3];
  const int k = (h & 7) >> 1;
  const uint32_t w = k == 0 ? x.x : k == 1 ? x.y : k == 2 ? x.z : x.w;
  return make_float2(bf16_lo(w), bf16_hi(w));
}
template <>
__device__ __forceinline__ float2 pair_of<float>(const uint4 (&r)[4], int h) {
  const uint4 x = r[h >> 2];
  return (h & 3) == 0 ? make_float2(__uint_as_float(x.x), __uint_as_float(x.y))
                      : make_float2(__uint_as_float(x.z), __uint_as_float(x.w));
}

template <typename T>
__device__ __forceinline__ float2 diff2(float2 t, float2 d, float C);
template <>
__device__ __forceinline__ float2 diff2<uint16_t>(float2 t, float2 d, float C) {
  return __fadd2_rn(__fadd2_rn(t, make_float2(-d.x, -d.y)), make_float2(-C, -C));
}
template <>
__device__ __forceinline__ float2 diff2<float>(float2 t, float2 d, float C) {
  return make_float2(diff_ref<float>(t.x, d.x, C), diff_ref<float>(t.y, d.y, C));
}

// ---------------------------------------------------------------------------
// a1, warp-specialised stream (the launched path). Per CTA: 8 consumer warps,
// 1 TMA producer warp, 1 merger warp; 2 CTAs per SM; a 3-stage ring of 32 KB
// stages filled by 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx).
// Items q = (draft row r, chunk c) are swept in order, q = blockIdx.x + j*grid.
// No CTA-wide barrier in the loop:
//   * a consumer warp lifts its 1/8 of the chunk (t and d) into registers,
//     releases the stage (mbarrier `consumed`), takes its own reference
//     M = max t, C = M - max d (so e^{t-M} e^{-w} = e^{d - max d} <= 1: no
//     overflow for any input), accumulates S, A, D with packed FFMA2 math and
//     posts a warp partial (mbarriers `ready` / `freeb` guard the slot sets);
//   * the producer refills a stage as soon as it is consumed;
//   * the merger folds the 8 warp partials into the chunk partial in fp64
//     (same re-referencing as merge_row).
// ---------------------------------------------------------------------------
constexpr int kCWarps = 8;
constexpr int kWsThreads = 32 * (kCWarps + 2);  // + TMA producer warp + merger warp
#ifndef DSDE_WS_STAGES
#define DSDE_WS_STAGES 3
#endif
#ifndef DSDE_WS_CTAS
#define DSDE_WS_CTAS 2
#endif
constexpr int kWsStages = DSDE_WS_STAGES;  // stages per CTA
constexpr int kWsCtas = DSDE_WS_CTAS;      // CTAs per SM

struct WarpPartial {  // 24 bytes
  float S, A, D;      // about (M, C) of the warp slice
  float M, C, maxd;
};

template <typename T>
__host__ __device__ constexpr int stream_ws_smem() {
  return kWsStages * 2 * stage_row_bytes<T>() + kWsStages * 2 * kCWarps * (int)sizeof(WarpPartial) +
         6 * kWsStages * 8;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// q -> (draft row r, chunk c), advanced by the grid stride without divisions
struct ItemCursor {
  long long r;
  int c;
  __device__ void init(long long q, int nchunks) {
    r = q / nchunks;
    c = (int)(q - r * nchunks);
  }
  __device__ void advance(int dr, int dc, int nchunks) {
    r += dr;
    c += dc;
    if (c >= nchunks) {
      c -= nchunks;
      r += 1;
    }
  }
};

// Sequence of draft row r, by a warp-cooperative forward scan from `seq`
// (rows only move forward for a CTA): 32 cu_sl entries per round trip.
__device__ __forceinline__ int seq_of_row(const int32_t* cu_sl, int B, int seq, long long r) {
  const int lane = threadIdx.x & 31;
  while (true) {
    const int j = seq + 1 + lane;
    const bool le = j <= B - 1 && __ldg(cu_sl + j) <= r;  // sequence j starts at or before r
    const unsigned m = __ballot_sync(kFull, le);
    seq += __popc(m);
    if (m != kFull) return seq;
  }
}

template <typename T>
__device__ __forceinline__ void issue_item(const StreamTmaArgs& a, long long r, int c, int seq,
                                           uint8_t* dst, uint64_t* bar) {
  constexpr int CH = chunk_elems<T>(), ROWB = stage_row_bytes<T>();
  const int c0 = c * CH;
  const int n_el = min(CH, a.V - c0);
  const uint32_t bytes = (uint32_t)(n_el * (int)sizeof(T)) & ~15u;
  if (bytes) {
    mbar_arrive_expect_tx(bar, 2 * bytes);
    bulk_g2s(dst, reinterpret_cast<const T*>(a.tl) + (r + seq) * a.ld_t + c0, bytes, bar);
    bulk_g2s(dst + ROWB, reinterpret_cast<const T*>(a.dl) + r * a.ld_d + c0, bytes, bar);
  } else {
    mbar_arrive(bar);
  }
}

template <typename T>
__global__ void __launch_bounds__(kWsThreads, kWsCtas) k_stream_ws(StreamTmaArgs a) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, E = VEC * NV, CH = chunk_elems<T>();
  constexpr int ROWB = stage_row_bytes<T>();
  constexpr int SL = CH / kCWarps;  // elements of a chunk owned by one consumer warp
  extern __shared__ __align__(128) uint8_t smem[];
  WarpPartial* slots = reinterpret_cast<WarpPartial*>(smem + kWsStages * 2 * ROWB);
  uint64_t* full = reinterpret_cast<uint64_t*>(slots + kWsStages * 2 * kCWarps);
  uint64_t* consumed = full + kWsStages;
  uint64_t* ready = consumed + kWsStages;   // [stage][2]: 8 warp partials posted
  uint64_t* freeb = ready + 2 * kWsStages;  // [stage][2]: merger done with the slot set
  const long long n_items = (long long)a.total * a.nchunks;
  const int G = gridDim.x;
  const int dr = G / a.nchunks, dc = G % a.nchunks;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&consumed[s], kCWarps);
      for (int b = 0; b < 2; ++b) {
        mbar_init(&ready[2 * s + b], kCWarps);
        mbar_init(&freeb[2 * s + b], 1);
      }
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCWarps) {
    // ---------------- TMA producer: refill a stage once it is consumed ----------------
    // (the whole warp tracks the row -> sequence cursor; lane 0 issues the copies;
    // the next item's addresses are resolved before waiting for its stage)
    ItemCursor it;
    it.init(blockIdx.x, a.nchunks);
    int seq = 0;
    long long q = blockIdx.x;
    for (int s = 0; s < kWsStages && q < n_items; ++s, q += G) {
      seq = seq_of_row(a.cu_sl, a.B, seq, it.r);
      if (lane == 0) issue_item<T>(a, it.r, it.c, seq, smem + s * 2 * ROWB, &full[s]);
      it.advance(dr, dc, a.nchunks);
    }
    int s = 0;
    uint32_t round = 0;
    for (; q < n_items; q += G) {
      seq = seq_of_row(a.cu_sl, a.B, seq, it.r);
      mbar_wait(&consumed[s], round & 1u);
      if (lane == 0) {
        issue_item<T>(a, it.r, it.c, seq, smem + s * 2 * ROWB, &full[s]);
      }
      it.advance(dr, dc, a.nchunks);
      if (++s == kWsStages) {
        s = 0;
        ++round;
      }
    }
    return;
  }
  if (warp == kCWarps + 1) {
    // ---------------- merger: 8 warp partials -> chunk partial (fp64) ----------------
    int s = 0;
    uint32_t round = 0;
    for (long long q = blockIdx.x; q < n_items; q += G) {
      const uint32_t b = round & 1u, u = round >> 1;  // slot set (s, b), its u-th use
      mbar_wait(&ready[2 * s + b], u & 1u);
      const WarpPartial* wp = slots + (s * 2 + b) * kCWarps;
      float Mr = -INFINITY, Dx = -INFINITY;
#pragma unroll
      for (int w = 0; w < kCWarps; ++w) {
        Mr = fmaxf(Mr, wp[w].M);
        Dx = fmaxf(Dx, wp[w].maxd);
      }
      const WarpPartial p = wp[lane < kCWarps ? lane : 0];
      __syncwarp();
      if (lane == 0) mbar_arrive(&freeb[2 * s + b]);  // slot set reusable
      const float Cc = Mr - Dx;
      double S = 0.0, A = 0.0, D = 0.0;
      if (lane < kCWarps) {
        const double ls = (double)p.M - (double)Mr;  // -inf for an empty slice
        const double sc = exp(ls);
        const double dl = (double)p.C - (double)Cc;
        double sem, sg, E1;
        if (fabs(dl) < 1.0) {
          const double em = expm1(-dl);
          sem = sc * em;
          sg = sc * (em + dl);
          E1 = sc + sem;
        } else {
          E1 = exp(ls - dl);
          sem = E1 - sc;
          sg = sem + sc * dl;
        }
        S = sc * (double)p.S;
        A = sc * (double)p.A + sc * (double)p.S * dl;
        D = E1 * (double)p.D - (double)p.A * sem + (double)p.S * sg;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        S += __shfl_xor_sync(kFull, S, o);
        A += __shfl_xor_sync(kFull, A, o);
        D += __shfl_xor_sync(kFull, D, o);
      }
      if (lane == 0) {
        ChunkPartial cp;
        cp.S = S;
        cp.A = A;
        cp.D = D;
        cp.M = Mr;
        cp.C = Cc;
        cp.idx = 0;
        cp.flags = 0;
        cp.maxd = Dx;
        cp.pad = 0;
        a.part[q] = cp;
      }
      if (++s == kWsStages) {
        s = 0;
        ++round;
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  const float2 L2 = make_float2(kLog2e, kLog2e);
  // h(-w), h(u) = (e^u - 1 - u)/u^2, degree-7 Chebyshev fit on |u| <= 1
  // (1.1e-7 relative in fp32 Horner; tools/fit_g.py), in powers of w (odd
  // coefficients negated). The MUFU form is used only for |w| >= 1, where its
  // relative error 2^-21 e^|w| / g(w) stays below ~1e-6; a cut at 1/2 was
  // measured to push single-position KL errors to 1e-5.
  const float2 K7 = make_float2(-2.812654656736413e-06f, -2.812654656736413e-06f);
  const float2 K6 = make_float2(2.5358644052175805e-05f, 2.5358644052175805e-05f);
  const float2 K5 = make_float2(-1.9836986029986292e-04f, -1.9836986029986292e-04f);
  const float2 K4 = make_float2(1.3885394437238574e-03f, 1.3885394437238574e-03f);
  const float2 K3 = make_float2(-8.33334494382143e-03f, -8.33334494382143e-03f);
  const float2 K2 = make_float2(4.166673496365547e-02f, 4.166673496365547e-02f);
  const float2 K1 = make_float2(-1.666666716337204e-01f, -1.666666716337204e-01f);
  const float2 K0 = make_float2(0.5f, 0.5f);
  ItemCursor it;
  it.init(blockIdx.x, a.nchunks);
  int s = 0;
  uint32_t round = 0;
  for (long long q = blockIdx.x; q < n_items; q += G) {
    const int c0 = it.c * CH;
    const int n_el = min(CH, a.V - c0);
    mbar_wait(&full[s], round & 1u);
    const T* st = reinterpret_cast<const T*>(smem + s * 2 * ROWB);
    const T* sd = reinterpret_cast<const T*>(smem + s * 2 * ROWB + ROWB);
    // the lane's 2 x 16 words (raw bf16 pairs / fp32) of the chunk; converted
    // to fp32 pair by pair inside the statistics loop (low register pressure)
    uint4 rt[NV], rd[NV];
    float mt = -INFINITY, md = -INFINITY;
    if (n_el == CH) {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int e0 = warp * SL + (v * 32 + lane) * VEC;
        rt[v] = *reinterpret_cast<const uint4*>(st + e0);
        rd[v] = *reinterpret_cast<const uint4*>(sd + e0);
      }
    } else {
      // last chunk of a row: bulk-copied part from shared memory, an unaligned
      // tail (V * sizeof(T) not a multiple of 16) from global, padding after V
      const int bulk_el = (int)(((uint32_t)(n_el * (int)sizeof(T)) & ~15u) / sizeof(T));
      long long trow = 0;
      if (bulk_el < n_el) {
        int lo = 0, hi = a.B - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (__ldg(a.cu_sl + mid) <= it.r) lo = mid; else hi = mid - 1;
        }
        trow = it.r + lo;
      }
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int e0 = warp * SL + (v * 32 + lane) * VEC;
        T tb[VEC], db[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int idx = e0 + e;
          tb[e] = pad_bits<T>();
          db[e] = pad_bits<T>();
          if (idx < bulk_el) {
            tb[e] = st[idx];
            db[e] = sd[idx];
          } else if (idx < n_el) {
            tb[e] = reinterpret_cast<const T*>(a.tl)[trow * a.ld_t + c0 + idx];
            db[e] = reinterpret_cast<const T*>(a.dl)[it.r * a.ld_d + c0 + idx];
          }
        }
        rt[v] = *reinterpret_cast<const uint4*>(tb);
        rd[v] = *reinterpret_cast<const uint4*>(db);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&consumed[s]);
    if constexpr (sizeof(T) == 2) {
      // two independent max chains per row (short dependency chains)
      __nv_bfloat162 bt0 = *reinterpret_cast<const __nv_bfloat162*>(&rt[0].x), bt1 = bt0;
      __nv_bfloat162 bd0 = *reinterpret_cast<const __nv_bfloat162*>(&rd[0].x), bd1 = bd0;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const uint32_t wt[4] = {rt[v].x, rt[v].y, rt[v].z, rt[v].w};
        const uint32_t wd[4] = {rd[v].x, rd[v].y, rd[v].z, rd[v].w};
#pragma unroll
        for (int h = 0; h < 4; h += 2) {
          bt0 = __hmax2_nan(bt0, *reinterpret_cast<const __nv_bfloat162*>(&wt[h]));  // NaN propagates
          bt1 = __hmax2_nan(bt1, *reinterpret_cast<const __nv_bfloat162*>(&wt[h + 1]));
          bd0 = __hmax2(bd0, *reinterpret_cast<const __nv_bfloat162*>(&wd[h]));
          bd1 = __hmax2(bd1, *reinterpret_cast<const __nv_bfloat162*>(&wd[h + 1]));
        }
      }
      const __nv_bfloat162 bt = __hmax2_nan(bt0, bt1), bd = __hmax2(bd0, bd1);
      const float lo = __low2float(bt), hi = __high2float(bt);
      mt = (lo != lo || hi != hi) ? NAN : fmaxf(lo, hi);
      md = fmaxf(__low2float(bd), __high2float(bd));
    } else {
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const uint32_t wt[4] = {rt[v].x, rt[v].y, rt[v].z, rt[v].w};
        const uint32_t wd[4] = {rd[v].x, rd[v].y, rd[v].z, rd[v].w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          mt = max_nan(mt, __uint_as_float(wt[h]));
          md = fmaxf(md, __uint_as_float(wd[h]));
        }
      }
    }
    // warp reference: M = max t (NaN if any t is NaN), C = M - max d
    float M, Dmax;
    if constexpr (sizeof(T) == 2) {
      // both maxima are bf16 values: one packed shuffle chain
      __nv_bfloat162 pk = __floats2bfloat162_rn(mt, md);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t y = __shfl_xor_sync(kFull, *reinterpret_cast<const uint32_t*>(&pk), o);
        pk = __hmax2_nan(pk, *reinterpret_cast<const __nv_bfloat162*>(&y));
      }
      M = __low2float(pk);
      const float dh = __high2float(pk);
      Dmax = dh == dh ? dh : warp_max(md);  // all-NaN d in some lane: NaN-ignoring max
    } else {
      M = warp_max(mt);
      Dmax = warp_max(md);
    }
    if (__any_sync(kFull, mt != mt)) M = NAN;
    const uint32_t sb = round & 1u, su = round >> 1;  // slot set (s, sb), its su-th use
    WarpPartial p;
    if (M <= -1e30f) {  // slice beyond V (padding only): an empty partial (NaN is not empty)
      p.S = p.A = p.D = 0.f;
      p.M = -INFINITY;
      p.C = 0.f;
      p.maxd = -INFINITY;
    } else {
      const float Cw = M - Dmax;
      const float ML2 = M * kLog2e, DL2 = Dmax * kLog2e;
      const float2 nML2 = make_float2(-ML2, -ML2), nDL2 = make_float2(-DL2, -DL2);
      float2 S2 = make_float2(0.f, 0.f), A2 = S2, D2 = S2;
#ifdef DSDE_STREAM_LITE  // measurement experiment only: memory pipeline with minimal math
#pragma unroll
      for (int h = 0; h < E; h += 2) {
        const float2 tt = pair_of<T>(rt, h), dd = pair_of<T>(rd, h);
        S2 = __fadd2_rn(S2, tt);
        A2 = __fadd2_rn(A2, dd);
      }
#else
#pragma unroll
      for (int h = 0; h < E; h += 2) {
        const float2 tt = pair_of<T>(rt, h), dd = pair_of<T>(rd, h);
        const float2 xt = __ffma2_rn(tt, L2, nML2);
        const float2 arg = __ffma2_rn(dd, L2, nDL2);  // (d - max d) log2 e <= 0
        const float2 e = make_float2(fast_exp2(xt.x), fast_exp2(xt.y));
        const float2 f = make_float2(fast_exp2(arg.x), fast_exp2(arg.y));
        const float2 w = diff2<T>(tt, dd, Cw);
        // h(-w) by Estrin's scheme (dependency depth 4 instead of 7)
        const float2 w2 = __fmul2_rn(w, w);
        const float2 q01 = __ffma2_rn(K1, w, K0), q23 = __ffma2_rn(K3, w, K2);
        const float2 q45 = __ffma2_rn(K5, w, K4), q67 = __ffma2_rn(K7, w, K6);
        const float2 w4 = __fmul2_rn(w2, w2);
        const float2 q03 = __ffma2_rn(q23, w2, q01), q47 = __ffma2_rn(q67, w2, q45);
        const float2 pp = __ffma2_rn(q47, w4, q03);
        S2 = __fadd2_rn(S2, e);
        A2 = __ffma2_rn(e, w, A2);
        const float2 sm = __fmul2_rn(__fmul2_rn(e, w2), pp);
        const float2 bg = __ffma2_rn(e, w, __fadd2_rn(f, make_float2(-e.x, -e.y)));
        const float2 term =
            make_float2(fabsf(w.x) < 1.f ? sm.x : bg.x, fabsf(w.y) < 1.f ? sm.y : bg.y);
        D2 = __fadd2_rn(D2, term);
      }
#endif
      float S = S2.x + S2.y, A = A2.x + A2.y, D = D2.x + D2.y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        S += __shfl_xor_sync(kFull, S, o);
        A += __shfl_xor_sync(kFull, A, o);
        D += __shfl_xor_sync(kFull, D, o);
      }
      p.S = S;
      p.A = A;
      p.D = D;
      p.M = M;
      p.C = Cw;
      p.maxd = Dmax;
    }
    if (lane == 0) {
      if (su > 0) mbar_wait(&freeb[2 * s + sb], (su - 1) & 1u);
      slots[(s * 2 + sb) * kCWarps + warp] = p;
      mbar_arrive(&ready[2 * s + sb]);
    }
    it.advance(dr, dc, a.nchunks);
    if (++s == kWsStages) {
      s = 0;
      ++round;
    }
  }
}

// Merged statistics of one row about the row argmax.
struct RowStats {
  double M, C, S, A, D;
  int flags;
};

// fp64 merge of chunk partials in chunk order about the row reference
// M = max_c M_c and C = fp32(M - max_v d_v) (so every merged term
// e^{t-M} e^{-w} = e^{d - max d} <= 1; C is an fp32 value so the sampling
// pass can rebuild w exactly). Chunk c's w is shifted by Delta = C_c - C; with
// s = e^(M_c - M) and E1 = s e^-Delta:
//   S += s S_c,   A += s (A_c + S_c Delta),
//   D += E1 D_c - A_c s expm1(-Delta) + S_c s g(Delta),  g(x) = expm1(-x) + x.
__device__ RowStats merge_row(const ChunkPartial* P, int nchunks, bool pair) {
  float Mref = P[0].M, maxd = P[0].maxd;
  for (int c = 1; c < nchunks; ++c) {
    Mref = max_nan(Mref, P[c].M);
    maxd = fmaxf(maxd, P[c].maxd);
  }
  RowStats r;
  r.M = (double)Mref;
  r.C = pair ? (double)(Mref - maxd) : 0.0;
  r.S = r.A = r.D = 0.0;
  r.flags = 0;
  for (int c = 0; c < nchunks; ++c) {
    const ChunkPartial q = P[c];
    const double ls = (double)q.M - r.M;
    const double s = exp(ls);
    r.S += s * q.S;
    r.flags |= q.flags;
    if (pair) {
      const double dl = (double)q.C - r.C;
      double sem, sg, E1;  // s expm1(-dl), s g(dl), s e^-dl
      if (fabs(dl) < 1.0) {
        const double em = expm1(-dl);
        sem = s * em;
        sg = s * (em + dl);
        E1 = s + sem;
      } else {
        E1 = exp(ls - dl);
        sem = E1 - s;
        sg = sem + s * dl;
      }
      r.A += s * q.A + s * q.S * dl;
      r.D += E1 * q.D - q.A * sem + q.S * sg;
    }
  }
  return r;
}

struct FinArgs {
  int B, V, total, nchunks;
  const int32_t* cu_sl;
  const int32_t* tokens;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const uint64_t* seeds;
  const ChunkPartial* part;
  int32_t* acc_len;
  int32_t* emitted;
  float* kld;
  uint8_t* flags;
  SeqRec* rec;
  int* counter;
  int32_t* err;
};

// a2 + a3: one warp per sequence, lane j = draft position j (k_i <= 16 < 32);
// lane k_i also draws the uniforms of the bonus slot.
template <typename T>
__global__ void __launch_bounds__(128) k_finalize(FinArgs a) {
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= a.B) return;
  const int c0 = __ldg(a.cu_sl + i), c1 = __ldg(a.cu_sl + i + 1);
  const int k = c1 - c0;
  const bool range_ok = c0 >= 0 && k >= 1 && k <= DSDE_MAX_SL && c1 <= a.total;
  const bool rows_ok = (i != a.B - 1) || (c1 == a.total);
  if (!range_ok || !rows_ok) {
    if (lane == 0) {
      a.acc_len[i] = -1;
      a.rec[i].mode = MODE_ERROR;
      raise_device_error(a.err, range_ok ? DSDE_DERR_ROWS : DSDE_DERR_BAD_SL, i);
    }
    return;
  }
  const long long slot0 = (long long)c0 + i;
  double kl = 0.0, lr = 0.0, C = 0.0, lam = 0.0, M = 0.0;
  bool acc = false, near = false, bad_tok = false, nonfin = false;
  int rflags = 0;
  Uniforms u = {0.0, 0.0};
  if (lane <= k) u = philox_uniforms(__ldg(a.seeds + slot0 + lane));
  if (lane < k) {
    const long long drow = (long long)c0 + lane;
    const int x = __ldg(a.tokens + drow);
    bad_tok = x < 0 || x >= a.V;
    const RowStats r = merge_row(a.part + drow * a.nchunks, a.nchunks, true);
    rflags = r.flags;
    nonfin = !(isfinite(r.S) && isfinite(r.A) && isfinite(r.D) && r.S > 0.0 && isfinite(r.M) &&
               isfinite(r.C));
    // y = E_p[exp(-w)] - 1. KL = D/S + (log1p(y) - y) has no cancellation for
    // small KL; when y > 1 (the draft puts far more mass away from the
    // reference, e.g. disjoint supports) the equal form A/S + log1p(y) is used.
    const double y = (r.D - r.A) / r.S;
    lam = log1p(y);
    kl = fmax(0.0, y <= 1.0 ? r.D / r.S + (lam - y) : r.A / r.S + lam);
    C = r.C;
    M = r.M;
    if (!bad_tok) {
      const T* tp = reinterpret_cast<const T*>(a.tl) + (drow + i) * a.ld_t;
      const T* dp = reinterpret_cast<const T*>(a.dl) + drow * a.ld_d;
      const double tx = (double)load_logit<T>(tp + x), dx = (double)load_logit<T>(dp + x);
      lr = (tx - dx) - C + lam;
      nonfin |= !isfinite(lr);
    }
    const double pacc = lr >= 0.0 ? 1.0 : exp(lr);
    acc = u.acc < pacc;
    near = fabs(u.acc - pacc) < 1e-6;
  }
  const unsigned bt = __ballot_sync(kFull, bad_tok);
  const unsigned nf = __ballot_sync(kFull, nonfin);
  const unsigned am = __ballot_sync(kFull, acc);
  if (bt | nf) {
    if (lane < k) a.kld[c0 + lane] = NAN;
    if (lane <= k) {
      a.emitted[slot0 + lane] = DSDE_PAD;
      if (a.flags) a.flags[slot0 + lane] = 0;
    }
    if (lane == 0) {
      a.acc_len[i] = -1;
      a.rec[i].mode = MODE_ERROR;
      raise_device_error(a.err, bt ? DSDE_DERR_BAD_TOKEN : DSDE_DERR_NONFINITE, i);
    }
    return;
  }
  const int acc_run = __ffs(~am) - 1;  // first rejected lane (lanes >= k never accept)
  const int aa = acc_run < k ? acc_run : k;
  if (lane < k) a.kld[c0 + lane] = (float)kl;
  if (lane <= k) {
    a.emitted[slot0 + lane] = lane < aa ? __ldg(a.tokens + c0 + lane) : DSDE_PAD;
    if (a.flags) {
      uint8_t f = (uint8_t)(rflags & DSDE_FLAG_OVERFLOW);
      if (near && lane <= aa && lane < k) f |= DSDE_FLAG_ACCEPT_NEAR_TIE;
      a.flags[slot0 + lane] = f;
    }
  }
  if (lane == 0) {
    a.acc_len[i] = aa;
    a.counter[i] = 0;
  }
  if (lane == aa) {
    SeqRec r;
    r.slot = (int)(slot0 + aa);
    r.trow = slot0 + aa;
    r.u = u.smp;
    r.pad0 = 0;
    if (aa < k) {
      r.mode = MODE_RESIDUAL;
      r.drow = (long long)c0 + aa;
      r.M = (float)M;
      r.C = C;
      r.lam = lam;
    } else {
      r.mode = MODE_BONUS;
      r.drow = -1;
      r.M = 0.f;
      r.C = 0.0;
      r.lam = 0.0;
    }
    a.rec[i] = r;
  }
}

struct SampArgs {
  int B, V, nchunks, total;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const ChunkPartial* part;
  const SeqRec* rec;
  double* mass;
  int32_t* emitted;
  uint8_t* flags;
  float* cmax;
  int* counter;
  int32_t* err;
};


// ---------------------------------------------------------------------------
// a4: one launch for every draw of the step, warp-granular (no block barrier).
// Warp (i, u) forms the draw weights of sub-chunk u (SUB = 32*E elements,
// lane-strided 16-byte vectors) of sequence i and their mass; the last warp of
// sequence i to finish (atomic counter + threadfence) selects the token: an
// fp64 warp scan over the sub-chunk masses, then a warp scan inside the
// crossing sub-chunk (re-read from L2), in ascending token order (D7).
//   residual: rho_v = e_v (1 - exp(-z_v)) for z_v > 0, else 0, with
//             e_v = exp(t_v - M), z_v = w_v + lam, w_v = (t_v - d_v) - C exact,
//             lam added as hi + lo floats; 1 - exp(-z) = z (1 - z h(-z)) for
//             z < 1 (no cancellation), 1 - 2^(-z log2 e) otherwise;
//   bonus:    p_v up to a scale: exp(t_v - m_u) about the warp max m_u,
//             rescaled by exp(m_u - max_u m_u) in fp64 (one pass over the row).
// Every per-lane value is recomputed bit-identically by the select pass.
// ---------------------------------------------------------------------------
template <typename T>
__host__ __device__ constexpr int sub_elems() {
  return 32 * Traits<T>::VEC * Traits<T>::NV;
}

template <typename T>
__device__ __forceinline__ void load_vec(const T* row, int V, int e0, float* x) {
  constexpr int VEC = Traits<T>::VEC;
  if (e0 + VEC <= V) {
    unpack16<T>(*reinterpret_cast<const uint4*>(row + e0), x);
  } else {
#pragma unroll
    for (int e = 0; e < VEC; ++e) x[e] = (e0 + e < V) ? load_logit<T>(row + e0 + e) : -INFINITY;
  }
}

// Draw weights of this lane's elements of sub-chunk u: w[v*VEC + e] for token
// u*SUB + (v*32 + lane)*VEC + e. Returns the reference (residual: the row's M;
// bonus: the warp max of t over the sub-chunk, -inf if all padding).
template <typename T>
__device__ __forceinline__ float sub_weights(const SampArgs& a, const SeqRec& r, bool resid, int u,
                                             float (&w)[Traits<T>::VEC * Traits<T>::NV]) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, E = VEC * NV;
  const int lane = threadIdx.x & 31;
  const int base = u * sub_elems<T>() + lane * VEC;
  float t[E];
  const T* tp = reinterpret_cast<const T*>(a.tl) + r.trow * a.ld_t;
#pragma unroll
  for (int v = 0; v < NV; ++v) load_vec<T>(tp, a.V, base + v * 32 * VEC, t + v * VEC);
  if (resid) {
    float d[E];
    const T* dp = reinterpret_cast<const T*>(a.dl) + r.drow * a.ld_d;
#pragma unroll
    for (int v = 0; v < NV; ++v) load_vec<T>(dp, a.V, base + v * 32 * VEC, d + v * VEC);
    const float Cf = (float)r.C;  // exact: r.C holds an fp32 value
    const float lhi = (float)r.lam, llo = (float)(r.lam - (double)lhi);
    const float ML2 = r.M * kLog2e;
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const float ev = fast_exp2(fmaf(t[q], kLog2e, -ML2));  // 0 for padding (-inf)
      const float z = (diff_ref<T>(t[q], d[q], Cf) + lhi) + llo;
      float pz = -2.812654656736413e-06f;  // h(-z): tools/fit_g.py (degree 7, |u| <= 1)
      pz = fmaf(pz, z, 2.5358644052175805e-05f);
      pz = fmaf(pz, z, -1.9836986029986292e-04f);
      pz = fmaf(pz, z, 1.3885394437238574e-03f);
      pz = fmaf(pz, z, -8.33334494382143e-03f);
      pz = fmaf(pz, z, 4.166673496365547e-02f);
      pz = fmaf(pz, z, -1.666666716337204e-01f);
      pz = fmaf(pz, z, 0.5f);
      const float one_m = z < 1.f ? z * fmaf(-z, pz, 1.f) : 1.f - fast_exp2(-z * kLog2e);
      w[q] = (z > 0.f && ev > 0.f) ? ev * one_m : 0.f;
    }
    return r.M;
  }
  float m = -INFINITY;
#pragma unroll
  for (int q = 0; q < E; ++q) m = max_nan(m, t[q]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max_nan(m, __shfl_xor_sync(kFull, m, o));
  const float mL2 = m * kLog2e;
#pragma unroll
  for (int q = 0; q < E; ++q) w[q] = m == -INFINITY ? 0.f : fast_exp2(fmaf(t[q], kLog2e, -mL2));
  return m;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ double warp_incl_scan(double x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

template <typename T>
__global__ void __launch_bounds__(kThreads) k_sample(SampArgs a) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, E = VEC * NV, SUB = sub_elems<T>();
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const int nsub = (a.V + SUB - 1) / SUB;
  if (gw >= (long long)a.B * nsub) return;
  const int i = (int)(gw / nsub), u = (int)(gw - (long long)i * nsub);
  const SeqRec r = a.rec[i];
  if (r.mode != MODE_RESIDUAL && r.mode != MODE_BONUS) return;
  const bool resid = r.mode == MODE_RESIDUAL;
  double* wmass = a.mass + (long long)i * a.nchunks * kCWarps;
  float* wmax = a.cmax + (long long)i * a.nchunks * kCWarps;

  float w[E];
  const float mu = sub_weights<T>(a, r, resid, u, w);
  double m = 0.0;  // sub-chunk mass about its reference, in the select pass's order
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += w[v * VEC + e];
    m += warp_sum_d((double)ls);
  }
  int last = 0;
  if (lane == 0) {
    wmass[u] = m;
    wmax[u] = mu;
    __threadfence();
    last = atomicAdd(a.counter + i, 1) == nsub - 1;
  }
  if (!__shfl_sync(kFull, last, 0)) return;
  __threadfence();

  // ---- last warp of sequence i: select the token ----
  float Mg = -INFINITY;
  if (!resid) {
    for (int s0 = lane; s0 < nsub; s0 += 32) Mg = max_nan(Mg, __ldcg(wmax + s0));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mg = max_nan(Mg, __shfl_xor_sync(kFull, Mg, o));
  }
  auto scale_of = [&](int s0) -> double {  // sub-chunk mass scale to the common reference
    if (resid) return 1.0;
    const float ms = __ldcg(wmax + s0);
    return ms == -INFINITY ? 0.0 : exp((double)ms - (double)Mg);
  };
  double R = 0.0;
  for (int s0 = lane; s0 < nsub; s0 += 32) R += scale_of(s0) * __ldcg(wmass + s0);
  R = warp_sum_d(R);
  uint8_t fl = 0;
  if (!(R > 0.0) || !isfinite(R)) {
    if (lane == 0) {
      // residual mass 0 (p <= q everywhere in fp32; D7 fallback) or a
      // non-finite bonus row: no valid draw from these weights
      if (resid && isfinite(R)) {
        // D7: draw from p of the same target row (slow path, one lane)
        const float M = r.M;
        double tot = 0.0;
        for (int v = 0; v < a.V; ++v)
          tot += exp((double)load_logit<T>(reinterpret_cast<const T*>(a.tl) + r.trow * a.ld_t + v) - M);
        const double target = r.u * tot;
        double cum = 0.0;
        int tok = 0;
        for (int v = 0; v < a.V; ++v) {
          const double wv = exp((double)load_logit<T>(reinterpret_cast<const T*>(a.tl) + r.trow * a.ld_t + v) - M);
          cum += wv;
          if (wv > 0.0) tok = v;
          if (wv > 0.0 && cum > target) break;
        }
        a.emitted[r.slot] = tok;
        if (a.flags) a.flags[r.slot] |= DSDE_FLAG_FALLBACK;
      } else {
        a.emitted[r.slot] = DSDE_PAD;
        raise_device_error(a.err, DSDE_DERR_NONFINITE, i);
      }
    }
    return;
  }
  const double target = r.u * R;
  // crossing sub-chunk: first u with prefix(u) > target (fallback: last with mass)
  int us = -1, ulast = -1;
  double base = 0.0, base_last = 0.0, cum = 0.0;
  for (int g = 0; g < nsub; g += 32) {
    const int s0 = g + lane;
    const double ms = s0 < nsub ? scale_of(s0) * __ldcg(wmass + s0) : 0.0;
    const double incl = warp_incl_scan(ms, lane);
    const unsigned pos = __ballot_sync(kFull, ms > 0.0);
    const unsigned cross = __ballot_sync(kFull, ms > 0.0 && cum + incl > target);
    if (pos) {
      const int lp = 31 - __clz(pos);
      ulast = g + lp;
      base_last = cum + __shfl_sync(kFull, incl - ms, lp);
    }
    if (cross) {
      const int lc = __ffs(cross) - 1;
      us = g + lc;
      base = cum + __shfl_sync(kFull, incl - ms, lc);
      break;
    }
    cum += __shfl_sync(kFull, incl, 31);
  }
  if (us < 0) {
    us = ulast;
    base = base_last;
    fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
  }
  const double f = scale_of(us);
  if (us != u) sub_weights<T>(a, r, resid, us, w);
  int tok = -1;
  double lo = 0.0, hi = 0.0;
  int last_pos = -1;
  double lp_lo = 0.0, lp_hi = 0.0;
  double vbase = base;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += w[v * VEC + e];
    const double incl = warp_incl_scan((double)ls, lane);
    const double pre = vbase + f * (incl - (double)ls);
    int cand = -1;
    double clo = 0.0, chi = 0.0;
    float run = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float before = run;
      run += w[v * VEC + e];
      const double cb = pre + f * (double)before, ca = pre + f * (double)run;
      if (cand < 0 && w[v * VEC + e] > 0.f && ca > target) {
        cand = e;
        clo = cb;
        chi = ca;
      }
    }
    const unsigned bc = __ballot_sync(kFull, cand >= 0);
    const int tok_base = us * SUB + v * 32 * VEC;
    if (bc) {
      const int lc = __ffs(bc) - 1;
      tok = tok_base + lc * VEC + __shfl_sync(kFull, cand, lc);
      lo = __shfl_sync(kFull, clo, lc);
      hi = __shfl_sync(kFull, chi, lc);
      break;
    }
    // remember the last positive-weight token for the rounding corner
    int lpos = -1;
    double llo = 0.0, lhi = 0.0;
    {
      float run2 = 0.f;
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        const float before = run2;
        run2 += w[v * VEC + e];
        if (w[v * VEC + e] > 0.f) {
          lpos = e;
          llo = pre + f * (double)before;
          lhi = pre + f * (double)run2;
        }
      }
    }
    const unsigned bp = __ballot_sync(kFull, lpos >= 0);
    if (bp) {
      const int lp = 31 - __clz(bp);
      last_pos = tok_base + lp * VEC + __shfl_sync(kFull, lpos, lp);
      lp_lo = __shfl_sync(kFull, llo, lp);
      lp_hi = __shfl_sync(kFull, lhi, lp);
    }
    vbase += f * __shfl_sync(kFull, incl, 31);
  }
  if (tok < 0) {  // rounding corner: u R within rounding of the sub-chunk total
    tok = last_pos;
    lo = lp_lo;
    hi = lp_hi;
    fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
  }
  if (lane == 0) {
    if (fabs(r.u - lo / R) < 1e-6 || fabs(r.u - hi / R) < 1e-6) fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
    a.emitted[r.slot] = tok < 0 ? 0 : tok;
    if (a.flags) a.flags[r.slot] |= fl;
  }
}

#include "verify_fused.cuh"

template <typename T>
cudaError_t launch_verify(int B, int V, int total, const int32_t* cu_sl, const int32_t* tokens,
                          const void* tl, int64_t ld_t, const void* dl, int64_t ld_d,
                          const uint64_t* seeds, int32_t* acc_len, int32_t* emitted, float* kld,
                          uint8_t* flags, const VerifyWs& ws, int32_t* err, cudaStream_t s) {
  const int nc = (V + chunk_elems<T>() - 1) / chunk_elems<T>();
  if (getenv("DSDE_LEGACY_VERIFY") == nullptr) {
    // one persistent, cooperative launch for a1-a4 (verify_fused.cuh)
    constexpr int smem = fused_smem<T>();
    static int grid_per_dev[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    int& grid = grid_per_dev[dev & 63];
    if (grid == 0) {
      cudaFuncSetAttribute(k_verify_fused<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int sms = 148, per_sm = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_verify_fused<T>, kFzThreads, smem);
      grid = std::max(1, std::min(per_sm, kWsCtas)) * sms;
    }
    // draw items of a sequence are placed `lag` sequence blocks after its
    // stream items (all at the end by default: no pipeline waits on finalize)
    int lag = B;
    if (const char* e = getenv("DSDE_LAG")) lag = atoi(e) > 0 ? atoi(e) : B;
    lag = std::max(1, std::min(lag, B));
    cudaMemsetAsync(ws.counter, 0, sizeof(int) * (3 * (size_t)B + 2), s);
    cudaMemsetAsync(ws.counter + 3 * (size_t)B + 2, 0xff, sizeof(int) * 2 * (size_t)B, s);
    const int exp_flags = getenv("DSDE_EXP_FLAGS") ? atoi(getenv("DSDE_EXP_FLAGS")) : 0;
    FusedArgs fa{B, V, nc, total, lag, exp_flags, cu_sl, tokens, tl, ld_t, dl, ld_d, seeds, acc_len, emitted,
                 kld, flags, ws.part, ws.rec, ws.mass, ws.cmax, ws.counter,
                 ws.counter + 3 * (size_t)B + 2, err};
    void* args[] = {&fa};
    return cudaLaunchCooperativeKernel((const void*)k_verify_fused<T>, dim3(grid), dim3(kFzThreads),
                                       args, smem, s);
  }
  // legacy three-launch path (kept for A/B measurements)
  if (total > 0) {
    static bool attr_set = false;
    constexpr int smem = stream_ws_smem<T>();
    if (!attr_set) {
      cudaFuncSetAttribute(k_stream_ws<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr_set = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long items = (long long)total * nc;
    const int grid = (int)std::min<long long>(items, (long long)kWsCtas * sms);
    StreamTmaArgs ta{tl, ld_t, dl, ld_d, cu_sl, B, V, nc, total, ws.part};
    k_stream_ws<T><<<grid, kWsThreads, smem, s>>>(ta);
  }
  FinArgs fa{B, V, total, nc, cu_sl, tokens, tl, ld_t, dl, ld_d, seeds, ws.part,
             acc_len, emitted, kld, flags, ws.rec, ws.counter, err};
  k_finalize<T><<<(B + 3) / 4, 128, 0, s>>>(fa);
  SampArgs pa{B, V, nc, total, tl, ld_t, dl, ld_d, ws.part, ws.rec, ws.mass, emitted, flags,
              ws.cmax, ws.counter, err};
  const long long warps = (long long)B * ((V + sub_elems<T>() - 1) / sub_elems<T>());
  k_sample<T><<<(unsigned)((warps + kThreads / 32 - 1) / (kThreads / 32)), kThreads, 0, s>>>(pa);
  return cudaGetLastError();
}

}  // namespace dsde

using namespace dsde;

extern "C" size_t dsde_verify_workspace_size(int B, int total_draft_rows, int V, dsde_dtype dtype) {
  if (B < 1 || V < 2 || total_draft_rows < 0) return 0;
  return ws_layout(B, total_draft_rows, V, dtype, nullptr, nullptr);
}

extern "C" dsde_status dsde_verify(int B, int V, dsde_dtype dtype, int total_draft_rows,
                                   const int32_t* cu_sl, const int32_t* draft_tokens,
                                   const void* target_logits, int64_t ld_t,
                                   const void* draft_logits, int64_t ld_d,
                                   const uint64_t* seeds, int32_t* accepted_len,
                                   int32_t* emitted_tokens, float* kld, uint8_t* flags,
                                   void* workspace, size_t ws_bytes, dsde_state st, void* stream) {
  if (!st || !cu_sl || !draft_tokens || !target_logits || !draft_logits || !seeds ||
      !accepted_len || !emitted_tokens || !kld || !workspace)
    return DSDE_ERR_ARG;
  if (B < 1 || V < 2 || total_draft_rows < B || total_draft_rows > B * DSDE_MAX_SL)
    return DSDE_ERR_ARG;
  if (dtype != DSDE_F32 && dtype != DSDE_BF16) return DSDE_ERR_ARG;
  if (ld_t < V || ld_d < V) return DSDE_ERR_ARG;
  const size_t esz = dtype == DSDE_BF16 ? 2 : 4;
  if ((((uintptr_t)target_logits) | ((uintptr_t)draft_logits)) & 15) return DSDE_ERR_ARG;
  if (((size_t)ld_t * esz) % 16 || ((size_t)ld_d * esz) % 16) return DSDE_ERR_ARG;
  if (((uintptr_t)workspace) & 255) return DSDE_ERR_ARG;
  const size_t need = ws_layout(B, total_draft_rows, V, dtype, nullptr, nullptr);
  if (ws_bytes < need) return DSDE_ERR_ARG;
  const int nc = n_chunks(V, dtype);
  if ((long long)(total_draft_rows + B) * nc > 0x7fffffffLL) return DSDE_ERR_ARG;
  VerifyWs ws;
  ws_layout(B, total_draft_rows, V, dtype, &ws, reinterpret_cast<char*>(workspace));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (dtype == DSDE_BF16)
    e = launch_verify<uint16_t>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                                draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld,
                                flags, ws, st->err, s);
  else
    e = launch_verify<float>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                             draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld, flags,
                             ws, st->err, s);
  return e == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}
