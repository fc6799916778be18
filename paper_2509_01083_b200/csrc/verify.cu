// verify.cu — dsde_verify: the fused speculative-verification pass (§8(a) a1-a4).
//
// Pipeline (all on the caller's stream, no host synchronisation; 4 launches):
//   1. k_stream_ws   persistent warp-specialised CTAs, TMA-bulk ring: one streaming
//                    read of every (draft position row, vocab chunk) of the target
//                    and draft logits; S = sum e_v, A = sum e_v w_v, D = sum e_v g(w_v)
//                    about the chunk reference (a1).
//   2. k_finalize    one CTA per sequence, one warp per position: fp64 merge of the
//                    chunk partials, KL, log p/q; the Philox accept test, the first
//                    rejection a_i, token layout, the draw record (a2-a3).
//   3. k_draw_ws     same TMA ring over (sequence, chunk) of the drawn row: the mass
//                    of max(0, p - q) (row a_i) or of p (bonus row k_i) per sub-chunk.
//   4. k_select      one warp per sequence: the smallest token with C_v > u R (a4, D7).
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

#include "verify_draw.cuh"

template <typename T>
cudaError_t launch_verify(int B, int V, int total, const int32_t* cu_sl, const int32_t* tokens,
                          const void* tl, int64_t ld_t, const void* dl, int64_t ld_d,
                          const uint64_t* seeds, int32_t* acc_len, int32_t* emitted, float* kld,
                          uint8_t* flags, const VerifyWs& ws, int32_t* err, Profiler* prof,
                          cudaStream_t s) {
  const bool pr = prof != nullptr && prof->on;
  auto mark = [&]() {
    if (pr) cudaEventRecord(prof->next(), s);
  };
  mark();
  const int nc = (V + chunk_elems<T>() - 1) / chunk_elems<T>();
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static bool attr_set[64] = {false};
  if (!attr_set[dev & 63]) {
    cudaFuncSetAttribute(k_stream_ws<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, stream_ws_smem<T>());
    cudaFuncSetAttribute(k_draw_ws<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, draw_ws_smem<T>());
    attr_set[dev & 63] = true;
  }
  // a1: statistics of every (draft row, vocab chunk)
  if (total > 0) {
    const long long items = (long long)total * nc;
    const int grid = (int)std::min<long long>(items, (long long)kWsCtas * sms);
    StreamTmaArgs ta{tl, ld_t, dl, ld_d, cu_sl, B, V, nc, total, ws.part};
    k_stream_ws<T><<<grid, kWsThreads, stream_ws_smem<T>(), s>>>(ta);
  }
  mark();
  // a2-a3: row merge, KL, accept test, layout, draw record
  FinArgs fa{B, V, total, nc, cu_sl, tokens, tl, ld_t, dl, ld_d, seeds, ws.part,
             acc_len, emitted, kld, flags, ws.rec, err};
  k_finalize<T><<<B, kFinThreads, 0, s>>>(fa);
  mark();
  // a4: draw-weight masses of the drawn rows, then the inverse-CDF select
  {
    const long long items = (long long)B * nc;
    const int grid = (int)std::min<long long>(items, (long long)kWsCtas * sms);
    DrawArgs da{B, V, nc, tl, ld_t, dl, ld_d, ws.rec, ws.mass, ws.cmax};
    k_draw_ws<T><<<grid, kDrawThreads, draw_ws_smem<T>(), s>>>(da);
  }
  mark();
  SelArgs sa{B, V, nc, tl, ld_t, dl, ld_d, ws.rec, ws.mass, ws.cmax, emitted, flags, err};
  k_select<T><<<(B + 3) / 4, 128, 0, s>>>(sa);
  mark();
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
                                flags, ws, st->err, st->prof, s);
  else
    e = launch_verify<float>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                             draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld, flags,
                             ws, st->err, st->prof, s);
  return e == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}
