// verify.cu — dsde_verify / dsde_step: the speculative-verification pass
// (§8(a) a1-a4; with dsde_step also a5-a7).
//
// Default pipeline (all on the caller's stream, no host synchronisation; 2 launches):
//   1. k_stream_ldg  one streaming read of every (draft position row, vocab slice)
//                    of the target and draft logits; per 2048-token (bf16) /
//                    512-token (fp32) slice: S = sum e_v, A = sum e_v w_v,
//                    D = sum e_v g(w_v) about the slice reference (a1).
//   2. k_tail        one CTA per sequence (verify_draw.cuh): fp64 merge of the
//                    slice partials, KL, log p/q, the Philox accept test, the
//                    first rejection a_i and token layout (a2-a3); the draw-weight
//                    masses of the drawn row (residual row a_i or bonus row k_i)
//                    and the inverse-CDF select (a4); in dsde_step also the
//                    signal / SL^ (a5-a6) and the batch cap (a7).
// Variants kept for A/B measurement (env, read once per process):
// DSDE_STREAM=tma (TMA producer warp + 8 consumer warps, CTA shared-memory
// ring), DSDE_TAIL=split (k_finalize, k_draw_ldg, k_select) and DSDE_TAIL=fused
// (one persistent kernel for the whole step, verify_fused.cuh). DESIGN.md §8
// lists their measurements.
//
// Numerics: with e_v = exp(t_v - M), w_v = (t_v - d_v) - C, C = M - max d
// (an fp32 value), and g(w) = exp(-w) - 1 + w >= 0:
//   KL(p||q) = D/S + (log1p(y) - y),  y = (D - A)/S = E_p[exp(-w)] - 1,
//   log p(x)/q(x) = (t_x - d_x) - C + log1p(y),
//   q_v / p_v = exp(-(w_v + log1p(y))).
// D sums non-negative terms, so the small-KL regime has no cancellation (the naive
// E_p[t - d] - LSE_t + LSE_d form loses ~1e-3 relative at KL ~ 1e-3).
// e_v e^{-w_v} = e^{d_v - max d} <= 1, so no term overflows for any finite input.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cuda_bf16.h>

#include "common.cuh"
#include "state.cuh"
#include "signal.cuh"

namespace dsde {

template <typename T>
struct Traits;
#ifndef DSDE_NV_BF16
#define DSDE_NV_BF16 8
#endif
#ifndef DSDE_NVD_BF16
#define DSDE_NVD_BF16 4
#endif
template <>
struct Traits<uint16_t> {                  // bf16 bit patterns
  static constexpr int VEC = 8;            // elements per 16-byte vector
  static constexpr int NV = DSDE_NV_BF16;  // vectors per lane per row slice, a1 stream
  static constexpr int NVD = DSDE_NVD_BF16;  // the same for the a4 draw pass
};
template <>
struct Traits<float> {
  static constexpr int VEC = 4;
  static constexpr int NV = 4;
  static constexpr int NVD = 4;
};
// one warp's slice of a row: 32 lanes x NV vectors x VEC elements (stream),
// 32 x NVD x VEC (draw)
template <typename T>
__host__ __device__ constexpr int sub_elems() {
  return 32 * Traits<T>::VEC * Traits<T>::NV;
}
template <typename T>
__host__ __device__ constexpr int sub_elems_d() {
  return 32 * Traits<T>::VEC * Traits<T>::NVD;
}
constexpr int kCWarps = 8;  // TMA variant: consumer warps per CTA = slices per stage
template <typename T>
__host__ __device__ constexpr int chunk_elems() {
  return kCWarps * sub_elems<T>();
}

// statistics of one row slice about its own reference (32 bytes)
struct SubPartial {
  float S, A, D;  // sum e, sum e w, sum e g(w), e = exp(t - M), w = (t - d) - C
  float M;        // slice max of t (-inf: padding only; NaN if any t is NaN)
  float C;        // M - maxd
  float maxd;     // slice max of d
  float pad0, pad1;
};
static_assert(sizeof(SubPartial) == 32, "SubPartial layout");

enum { MODE_NONE = 0, MODE_RESIDUAL = 1, MODE_BONUS = 2, MODE_ERROR = 3, MODE_ARGMAX = 4 };  // ARGMAX: greedy bonus row

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
  double S;          // sum_v exp(t_v - M) of the drawn row (residual)
};
static_assert(sizeof(SeqRec) == 64, "SeqRec layout");

struct VerifyWs {
  SubPartial* part;  // [total * nsub] slice statistics of every draft row
  SeqRec* rec;       // [B]
  double* mass;      // [B * nsub_d] draw-weight mass per draw slice of the drawn row
  float* ref;        // [B * nsub_d] reference of each slice mass (bonus)
  void* rowres;      // [total] per-row results of the fused kernel (48 B each)
  int* counters;     // fused kernel: ctl[8], row_cnt[total], seq_cnt/draw_cnt/fin/queue[B]
  size_t counter_bytes;
};

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

constexpr int kCtlInts = 128;  // the fused kernel's control block (FusedCtl), ints

// slices per row: exact for the warp-per-slice kernels; rounded up to whole
// 8-slice chunks for the TMA variant (the workspace is sized for the latter)
inline int n_subs(int V, dsde_dtype dt, bool chunked = true) {
  const int se = dt == DSDE_BF16 ? sub_elems<uint16_t>() : sub_elems<float>();
  if (!chunked) return (V + se - 1) / se;
  const int ce = kCWarps * se;
  return (V + ce - 1) / ce * kCWarps;
}

inline int n_subs_d(int V, dsde_dtype dt) {
  const int se = dt == DSDE_BF16 ? sub_elems_d<uint16_t>() : sub_elems_d<float>();
  return (V + se - 1) / se;
}

inline size_t ws_layout(int B, int total, int V, dsde_dtype dt, VerifyWs* ws, char* base) {
  const int ns = n_subs(V, dt), nd = n_subs_d(V, dt);
  const size_t p_bytes = align256(sizeof(SubPartial) * (size_t)total * ns);
  const size_t r_bytes = align256(sizeof(SeqRec) * (size_t)B);
  const size_t m_bytes = align256(sizeof(double) * (size_t)B * nd);
  const size_t x_bytes = align256(sizeof(float) * (size_t)B * nd);
  const size_t rr_bytes = align256((size_t)48 * total);
  const size_t c_bytes = align256(sizeof(int) * (kCtlInts + (size_t)total + 4 * (size_t)B));
  if (ws) {
    ws->part = reinterpret_cast<SubPartial*>(base);
    ws->rec = reinterpret_cast<SeqRec*>(base + p_bytes);
    ws->mass = reinterpret_cast<double*>(base + p_bytes + r_bytes);
    ws->ref = reinterpret_cast<float*>(base + p_bytes + r_bytes + m_bytes);
    ws->rowres = base + p_bytes + r_bytes + m_bytes + x_bytes;
    ws->counters = reinterpret_cast<int*>(base + p_bytes + r_bytes + m_bytes + x_bytes + rr_bytes);
    ws->counter_bytes = sizeof(int) * (kCtlInts + (size_t)total + 4 * (size_t)B);
  }
  return p_bytes + r_bytes + m_bytes + x_bytes + rr_bytes + c_bytes;
}

// max that propagates NaN (a NaN logit must reach the non-finite check)
__device__ __forceinline__ float max_nan(float a, float b) { return (b > a || b != b) ? b : a; }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
  return v;
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

template <typename T>
__device__ __forceinline__ T pad_bits();
template <>
__device__ __forceinline__ uint16_t pad_bits<uint16_t>() { return (uint16_t)0xF14Au; }  // bf16 ~ -1e30
template <>
__device__ __forceinline__ float pad_bits<float>() { return -1e30f; }

// Elements h, h+1 (h even) of a lane's N x 16-byte vectors as an fp32 pair.
template <typename T, int N>
__device__ __forceinline__ float2 pair_of(const uint4 (&r)[N], int h) {
  if constexpr (sizeof(T) == 2) {
    const uint4 x = r[h >> 3];
    const int k = (h & 7) >> 1;
    const uint32_t w = k == 0 ? x.x : k == 1 ? x.y : k == 2 ? x.z : x.w;
    return make_float2(bf16_lo(w), bf16_hi(w));
  } else {
    const uint4 x = r[h >> 2];
    return (h & 3) == 0 ? make_float2(__uint_as_float(x.x), __uint_as_float(x.y))
                        : make_float2(__uint_as_float(x.z), __uint_as_float(x.w));
  }
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
// Loading a lane's words of row slice u: token u*SUB + (v*32 + lane)*VEC + e.
// Full slices use 128-bit loads; the last slice of a row pads past V with a
// value whose weights are exactly 0.
// ---------------------------------------------------------------------------
template <typename T, int NV>
__device__ __forceinline__ void load_slice(const T* row, int V, int u, uint4 (&r)[NV]) {
  constexpr int VEC = Traits<T>::VEC, SUB = 32 * VEC * NV;
  const int lane = threadIdx.x & 31;
  if ((u + 1) * SUB <= V) {
#pragma unroll
    for (int v = 0; v < NV; ++v) r[v] = ld_stream_v4(row + u * SUB + (v * 32 + lane) * VEC);
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int e0 = u * SUB + (v * 32 + lane) * VEC;
      if (e0 + VEC <= V) {
        r[v] = ld_stream_v4(row + e0);
      } else {
        T b[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) b[e] = (e0 + e < V) ? row[e0 + e] : pad_bits<T>();
        r[v] = *reinterpret_cast<const uint4*>(b);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// a1 per warp slice: reference M = max t (NaN if any t is NaN), C = M - max d,
// then S, A, D with packed FFMA2 math. g(w) for |w| < 1 is w^2 h(-w) with
// h(u) = (e^u - 1 - u)/u^2 as a degree-6 Chebyshev fit on |u| <= 1 (2.0e-7
// relative in fp32 Horner; `tools/fit_g.py --deg 6`) in powers of w (odd
// coefficients negated; DSDE_POLY_DEG7 selects the 1.1e-7 degree-7 fit);
// for |w| >= 1 it is f - e + e w with f = e^{d - max d} from MUFU.EX2, whose
// relative error 2^-21 e^|w| / g(w) stays below ~1e-6 there (a cut at 1/2 was
// measured to push single-position KL errors to 1e-5).
// ---------------------------------------------------------------------------
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// Lane-level running maxima of t (NaN-propagating) and d over 16-byte vectors.
template <typename T>
struct LaneMax {
  __nv_bfloat162 bt0, bt1, bd0, bd1;  // bf16: two packed chains per row
  float mt, md;                       // fp32
  __device__ __forceinline__ void init() {
    const __nv_bfloat162 ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    bt0 = bt1 = bd0 = bd1 = ninf;
    mt = md = -INFINITY;
  }
  __device__ __forceinline__ void add(const uint4& t, const uint4& d) {
    const uint32_t wt[4] = {t.x, t.y, t.z, t.w};
    const uint32_t wd[4] = {d.x, d.y, d.z, d.w};
    if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int h = 0; h < 4; h += 2) {
        bt0 = __hmax2_nan(bt0, *reinterpret_cast<const __nv_bfloat162*>(&wt[h]));  // NaN propagates
        bt1 = __hmax2_nan(bt1, *reinterpret_cast<const __nv_bfloat162*>(&wt[h + 1]));
        bd0 = __hmax2(bd0, *reinterpret_cast<const __nv_bfloat162*>(&wd[h]));
        bd1 = __hmax2(bd1, *reinterpret_cast<const __nv_bfloat162*>(&wd[h + 1]));
      }
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        mt = max_nan(mt, __uint_as_float(wt[h]));
        md = fmaxf(md, __uint_as_float(wd[h]));
      }
    }
  }
  // warp-wide slice reference: M = max t (NaN if any t is NaN), Dmax = max d
  __device__ __forceinline__ void reduce(float& M, float& Dmax) {
    if constexpr (sizeof(T) == 2) {
      const __nv_bfloat162 bt = __hmax2_nan(bt0, bt1), bd = __hmax2(bd0, bd1);
      const float lo = __low2float(bt), hi = __high2float(bt);
      mt = (lo != lo || hi != hi) ? NAN : fmaxf(lo, hi);
      md = fmaxf(__low2float(bd), __high2float(bd));
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
  }
};

// Per-slice constants of the a1 sums about the reference (M, C = M - max d).
struct SumRef {
  float2 nML2, nDL2;
  float Cw;
  __device__ __forceinline__ SumRef(float M, float Dmax) {
    Cw = M - Dmax;
    const float ML2 = M * kLog2e, DL2 = Dmax * kLog2e;
    nML2 = make_float2(-ML2, -ML2);
    nDL2 = make_float2(-DL2, -DL2);
  }
};

// a1 accumulation of one element pair (packed FFMA2 math, two MUFU.EX2 per
// element): S += e, A += e w, D += e g(w).
// ENT (opt-in): also Sd += f and E += f (d - max d), f = e^{d - max d},
// the draft's own softmax sums about the slice max of d (H(q) = log Sd - E / Sd).
struct EntAcc {
  float2 Sd, E;
};

template <typename T, bool ENT = false>
__device__ __forceinline__ void pair_accum_w(float2 tt, float2 dd, float2 w, const SumRef& R, float2& S2,
                                             float2& A2, float2& D2, EntAcc* ent = nullptr) {
  const float2 L2 = make_float2(kLog2e, kLog2e);
#ifndef DSDE_POLY_DEG7
  const float2 K6 = make_float2(2.5358644052175805e-05f, 2.5358644052175805e-05f);
  const float2 K5 = make_float2(-2.0329201652202755e-04f, -2.0329201652202755e-04f);
  const float2 K4 = make_float2(1.3885394437238574e-03f, 1.3885394437238574e-03f);
  const float2 K3 = make_float2(-8.330884389579296e-03f, -8.330884389579296e-03f);
  const float2 K2 = make_float2(4.166673496365547e-02f, 4.166673496365547e-02f);
  const float2 K1 = make_float2(-1.6666696965694427e-01f, -1.6666696965694427e-01f);
  const float2 K0 = make_float2(0.5f, 0.5f);
#else
  const float2 K7 = make_float2(-2.812654656736413e-06f, -2.812654656736413e-06f);
  const float2 K6 = make_float2(2.5358644052175805e-05f, 2.5358644052175805e-05f);
  const float2 K5 = make_float2(-1.9836986029986292e-04f, -1.9836986029986292e-04f);
  const float2 K4 = make_float2(1.3885394437238574e-03f, 1.3885394437238574e-03f);
  const float2 K3 = make_float2(-8.33334494382143e-03f, -8.33334494382143e-03f);
  const float2 K2 = make_float2(4.166673496365547e-02f, 4.166673496365547e-02f);
  const float2 K1 = make_float2(-1.666666716337204e-01f, -1.666666716337204e-01f);
  const float2 K0 = make_float2(0.5f, 0.5f);
#endif
  const float2 xt = __ffma2_rn(tt, L2, R.nML2);
  const float2 arg = __ffma2_rn(dd, L2, R.nDL2);  // (d - max d) log2 e <= 0
  const float2 e = make_float2(fast_exp2(xt.x), fast_exp2(xt.y));
  const float2 f = make_float2(fast_exp2(arg.x), fast_exp2(arg.y));
  const float2 w2 = __fmul2_rn(w, w);
#ifndef DSDE_POLY_DEG7
  float2 pp = __ffma2_rn(K6, w, K5);
#else
  float2 pp = __ffma2_rn(K7, w, K6);
  pp = __ffma2_rn(pp, w, K5);
#endif
  pp = __ffma2_rn(pp, w, K4);
  pp = __ffma2_rn(pp, w, K3);
  pp = __ffma2_rn(pp, w, K2);
  pp = __ffma2_rn(pp, w, K1);
  pp = __ffma2_rn(pp, w, K0);
  S2 = __fadd2_rn(S2, e);
  A2 = __ffma2_rn(e, w, A2);
  const float2 sm = __fmul2_rn(__fmul2_rn(e, w2), pp);
  const float2 bg = __ffma2_rn(e, w, __fadd2_rn(f, make_float2(-e.x, -e.y)));
  const float2 term = make_float2(fabsf(w.x) < 1.f ? sm.x : bg.x, fabsf(w.y) < 1.f ? sm.y : bg.y);
  D2 = __fadd2_rn(D2, term);
  if constexpr (ENT) {
    ent->Sd = __fadd2_rn(ent->Sd, f);
    ent->E = __ffma2_rn(f, __fmul2_rn(arg, make_float2(kLn2, kLn2)), ent->E);
  }
}

template <typename T, bool ENT = false>
__device__ __forceinline__ void pair_accum(float2 tt, float2 dd, const SumRef& R, float2& S2, float2& A2,
                                           float2& D2, EntAcc* ent = nullptr) {
  pair_accum_w<T, ENT>(tt, dd, diff2<T>(tt, dd, R.Cw), R, S2, A2, D2, ent);
}

// The sums of one 16-byte vector pair. When every |w| of the vector is below 2
// in every lane of the warp (the common case once the draft tracks the target),
// g(w) = w^2 h(-w) is a single degree-7 polynomial (Chebyshev fit of h on
// |u| <= 2, 2.1e-6 relative in fp32 Horner, `tools/fit_g.py --deg 7 --range 2`;
// DESIGN D19 — DSDE_WIDE_DEG=8 selects the 3.3e-7 degree-8 fit)
// and the e^{d - max d} exponential, the big-|w| form and the per-element
// select are skipped; otherwise every pair takes pair_accum (the test costs one
// FMNMX3 per pair; a slice-level "stop testing after a failure" flag and a
// separate untested path both measured slower on cfg3, faster only on cfg4).
#ifndef DSDE_WIDE_POLY
#define DSDE_WIDE_POLY 1
#endif
#ifndef DSDE_WIDE_DEG
#define DSDE_WIDE_DEG 7
#endif
template <typename T, bool ENT = false>
__device__ __forceinline__ void vec_accum(const uint4& t, const uint4& d, const SumRef& R, float2& S2,
                                          float2& A2, float2& D2, EntAcc* ent = nullptr) {
  constexpr int P = Traits<T>::VEC / 2;
  const uint4 rt[1] = {t}, rd[1] = {d};
#if DSDE_WIDE_POLY
  float2 tt[P], w[P];
  float am = 0.f;
#pragma unroll
  for (int h = 0; h < P; ++h) {
    tt[h] = pair_of<T>(rt, 2 * h);
    w[h] = diff2<T>(tt[h], pair_of<T>(rd, 2 * h), R.Cw);
    am = fmaxf(am, fmaxf(fabsf(w[h].x), fabsf(w[h].y)));
  }
  constexpr float kWideR = 2.f;
  if (__all_sync(kFull, am < kWideR)) {
    const float2 L2 = make_float2(kLog2e, kLog2e);
#pragma unroll
    for (int h = 0; h < P; ++h) {
      const float2 xt = __ffma2_rn(tt[h], L2, R.nML2);
      const float2 e = make_float2(fast_exp2(xt.x), fast_exp2(xt.y));
      const float2 ww = w[h];
      // h(-w) in powers of w (odd coefficients negated)
#if DSDE_WIDE_DEG == 7  // degree 7 on |u| <= 2 (2.1e-6 relative, the default)
      float2 pp = __ffma2_rn(make_float2(-2.990256007251446e-06f, -2.990256007251446e-06f), ww,
                             make_float2(2.7102691092295572e-05f, 2.7102691092295572e-05f));
      pp = __ffma2_rn(pp, ww, make_float2(-1.9769996288232505e-04f, -1.9769996288232505e-04f));
      pp = __ffma2_rn(pp, ww, make_float2(1.3830546522513032e-03f, 1.3830546522513032e-03f));
      pp = __ffma2_rn(pp, ww, make_float2(-8.334130048751831e-03f, -8.334130048751831e-03f));
      pp = __ffma2_rn(pp, ww, make_float2(4.167136549949646e-02f, 4.167136549949646e-02f));
      pp = __ffma2_rn(pp, ww, make_float2(-1.666664332151413e-01f, -1.666664332151413e-01f));
      pp = __ffma2_rn(pp, ww, make_float2(0.49999940395355225f, 0.49999940395355225f));
#else  // degree 8 on |u| <= 2 (3.3e-7 relative)
      float2 pp = __ffma2_rn(make_float2(2.972247159505059e-07f, 2.972247159505059e-07f), ww,
                             make_float2(-2.990256007251446e-06f, -2.990256007251446e-06f));
      pp = __ffma2_rn(pp, ww, make_float2(2.47248935920652e-05f, 2.47248935920652e-05f));
      pp = __ffma2_rn(pp, ww, make_float2(-1.9769996288232505e-04f, -1.9769996288232505e-04f));
      pp = __ffma2_rn(pp, ww, make_float2(1.388999167829752e-03f, 1.388999167829752e-03f));
      pp = __ffma2_rn(pp, ww, make_float2(-8.334130048751831e-03f, -8.334130048751831e-03f));
      pp = __ffma2_rn(pp, ww, make_float2(4.166661202907562e-02f, 4.166661202907562e-02f));
      pp = __ffma2_rn(pp, ww, make_float2(-1.666664332151413e-01f, -1.666664332151413e-01f));
      pp = __ffma2_rn(pp, ww, make_float2(0.5f, 0.5f));
#endif
      const float2 ew = __fmul2_rn(e, ww);
      S2 = __fadd2_rn(S2, e);
      A2 = __fadd2_rn(A2, ew);
      const float2 wh = __fmul2_rn(ww, pp);
      D2 = __ffma2_rn(ew, wh, D2);  // e w^2 h(-w)
      if constexpr (ENT) {
        // f = e e^{-w} = e (1 - w + w^2 h(-w)); d - max d = (t - M) - w
        const float2 f = __ffma2_rn(ew, __fadd2_rn(wh, make_float2(-1.f, -1.f)), e);
        const float2 dm = __ffma2_rn(xt, make_float2(kLn2, kLn2), make_float2(-ww.x, -ww.y));
        ent->Sd = __fadd2_rn(ent->Sd, f);
        ent->E = __ffma2_rn(f, dm, ent->E);
      }
    }
    return;
  }
#pragma unroll
  for (int h = 0; h < P; ++h) pair_accum_w<T, ENT>(tt[h], pair_of<T>(rd, 2 * h), w[h], R, S2, A2, D2, ent);
#else
#pragma unroll
  for (int h = 0; h < Traits<T>::VEC; h += 2)
    pair_accum<T, ENT>(pair_of<T>(rt, h), pair_of<T>(rd, h), R, S2, A2, D2, ent);
#endif
}

__device__ __forceinline__ SubPartial empty_partial() {
  SubPartial p;
  p.pad0 = p.pad1 = 0.f;
  p.S = p.A = p.D = 0.f;
  p.M = -INFINITY;
  p.C = 0.f;
  p.maxd = -INFINITY;
  return p;
}

__device__ __forceinline__ SubPartial finish_partial(float2 S2, float2 A2, float2 D2, float M, float Dmax,
                                                     float Cw) {
  float S = S2.x + S2.y, A = A2.x + A2.y, D = D2.x + D2.y;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_xor_sync(kFull, S, o);
    A += __shfl_xor_sync(kFull, A, o);
    D += __shfl_xor_sync(kFull, D, o);
  }
  SubPartial p;
  p.pad0 = p.pad1 = 0.f;
  p.S = S;
  p.A = A;
  p.D = D;
  p.M = M;
  p.C = Cw;
  p.maxd = Dmax;
  return p;
}

// `after_max` runs (warp-uniformly) once the slice maxima are reduced over the
// warp, i.e. once every lane's words have been consumed.
template <typename T, int NV, typename Hook = NoHook, bool ENT = false>
__device__ __forceinline__ SubPartial slice_stats(const uint4 (&rt)[NV], const uint4 (&rd)[NV],
                                                  Hook after_max = Hook()) {
  LaneMax<T> mx;
  mx.init();
#pragma unroll
  for (int v = 0; v < NV; ++v) mx.add(rt[v], rd[v]);
  float M, Dmax;
  mx.reduce(M, Dmax);
  after_max();
  if (M <= -1e30f) return empty_partial();  // slice beyond V (padding only; NaN is not empty)
  const SumRef R(M, Dmax);
  float2 S2 = make_float2(0.f, 0.f), A2 = S2, D2 = S2;
  if constexpr (ENT) {
    EntAcc ent{S2, S2};
#pragma unroll
    for (int v = 0; v < NV; ++v) vec_accum<T, true>(rt[v], rd[v], R, S2, A2, D2, &ent);
    SubPartial p = finish_partial(S2, A2, D2, M, Dmax, R.Cw);
    float Sd = ent.Sd.x + ent.Sd.y, E = ent.E.x + ent.E.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Sd += __shfl_xor_sync(kFull, Sd, o);
      E += __shfl_xor_sync(kFull, E, o);
    }
    p.pad0 = Sd;
    p.pad1 = E;
    return p;
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) vec_accum<T>(rt[v], rd[v], R, S2, A2, D2);
    return finish_partial(S2, A2, D2, M, Dmax, R.Cw);
  }
}

// lane 0 writes the whole 32-byte partial (so a release by lane 0 covers it)
__device__ __forceinline__ void store_partial(SubPartial* dst, const SubPartial& p) {
  if ((threadIdx.x & 31) == 0) {
    reinterpret_cast<float4*>(dst)[0] = make_float4(p.S, p.A, p.D, p.M);
    reinterpret_cast<float4*>(dst)[1] = make_float4(p.C, p.maxd, p.pad0, p.pad1);
  }
}

// Sequence of draft row r, by a warp-cooperative forward scan from `seq`
// (rows only move forward for a warp): 32 cu_sl entries per round trip.
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

struct StreamArgs {
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const int32_t* cu_sl;
  int B, V, nsub, total;  // total: Σk_i, or the row capacity when dev_rows
  SubPartial* part;
  int dev_rows;           // dsde_config.device_rows: Σk_i = cu_sl[B] (<= total), read here
};

// rows this launch streams: the host's Σk_i, or (device_rows) cu_sl[B] clamped
// to the capacity the grid and workspace were sized for
__device__ __forceinline__ int stream_rows(const StreamArgs& a) {
  return a.dev_rows ? min(max(__ldg(a.cu_sl + a.B), 0), a.total) : a.total;
}

// ---------------------------------------------------------------------------
// a1, "ldg" variant: persistent warps over the units q = (draft row r, slice u),
// q = global warp + j * (total warps). Each lane keeps the NEXT unit's 2 x 4
// 16-byte vectors in flight while it computes the current one (ping-pong
// register buffers, no shared memory, no block barriers).
// ---------------------------------------------------------------------------
constexpr int kLdgThreads = 256;
#ifndef DSDE_LDG_MINB
#define DSDE_LDG_MINB 3
#endif
#ifndef DSDE_EXPERIMENT
#define DSDE_EXPERIMENT 0
#endif

#ifndef DSDE_ENT_MINB
#define DSDE_ENT_MINB 2
#endif
// the entropy variant carries two more accumulators: 2 CTAs per SM (up to 128
// registers) instead of spilling at the 80-register cap of 3 CTAs per SM
template <typename T, bool DEV_ROWS, bool ENT = false>
__global__ void __launch_bounds__(kLdgThreads, ENT ? DSDE_ENT_MINB : DSDE_LDG_MINB) k_stream_ldg(StreamArgs a) {
  constexpr int NV = Traits<T>::NV;
  const int total = DEV_ROWS ? stream_rows(a) : a.total;
  const long long n_units = (long long)total * a.nsub;
  const long long W = (long long)gridDim.x * (kLdgThreads / 32);
  long long q = (long long)blockIdx.x * (kLdgThreads / 32) + (threadIdx.x >> 5);
  // let the tail kernel launch (programmatic dependent launch) and become
  // resident on SMs as this grid drains; it waits for our completion
  asm volatile("griddepcontrol.launch_dependents;");
  if (q >= n_units) return;
  int seq = 0;
  // (row r, slice u) of unit q advanced incrementally by W units per step
  int r = (int)((unsigned)q / (unsigned)a.nsub), u = (int)q - r * a.nsub;
  const int dr = (int)((unsigned long long)W / (unsigned)a.nsub), du = (int)(W - (long long)dr * a.nsub);
  while (r < total) {
    uint4 rt[NV], rd[NV];
#if DSDE_EXPERIMENT == 2  // measurement only: math without the loads
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t x = 0x3f803f80u ^ ((uint32_t)(r * 977 + u) * 2654435761u + v * 40503u + threadIdx.x) & 0x007f007fu;
      rt[v] = make_uint4(x, x ^ 0x10001u, x ^ 0x20002u, x ^ 0x30003u);
      rd[v] = make_uint4(x ^ 0x40004u, x ^ 0x50005u, x, x ^ 0x60006u);
    }
#else
    seq = seq_of_row(a.cu_sl, a.B, seq, r);
    load_slice<T>(reinterpret_cast<const T*>(a.tl) + (long long)(r + seq) * a.ld_t, a.V, u, rt);
    load_slice<T>(reinterpret_cast<const T*>(a.dl) + (long long)r * a.ld_d, a.V, u, rd);
#endif
    SubPartial* dst = a.part + ((long long)r * a.nsub + u);
#if DSDE_EXPERIMENT == 1  // measurement only: the loads without the math
    uint32_t acc = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v) acc ^= rt[v].x ^ rt[v].y ^ rt[v].z ^ rt[v].w ^ rd[v].x ^ rd[v].y ^ rd[v].z ^ rd[v].w;
    SubPartial p{};
    p.S = __uint_as_float(acc);
    store_partial(dst, p);
#else
    store_partial(dst, slice_stats<T, NV, NoHook, ENT>(rt, rd));
#endif
    u += du;
    r += dr;
    if (u >= a.nsub) {
      u -= a.nsub;
      ++r;
    }
  }
}

// ---------------------------------------------------------------------------
// mbarrier / TMA bulk-copy primitives (PTX)
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

// ---------------------------------------------------------------------------
// a1, "tma" variant: per CTA 1 TMA producer warp + 8 consumer warps, 2 CTAs per
// SM, a kTmaStages ring of (target, draft) chunk stages filled by 1-D bulk
// copies. Items q = (draft row r, chunk c) are swept q = blockIdx.x + j*grid;
// consumer warp w takes slice u = c*8 + w of the staged chunk, releases the
// stage, and writes its slice partial.
// ---------------------------------------------------------------------------
constexpr int kTmaThreads = 32 * (kCWarps + 1);
constexpr int kTmaStages = 3;
constexpr int kTmaCtas = 2;

template <typename T>
__host__ __device__ constexpr int stage_row_bytes() {
  return chunk_elems<T>() * (int)sizeof(T);
}
template <typename T>
__host__ __device__ constexpr int tma_smem() {
  return kTmaStages * 2 * stage_row_bytes<T>() + 16 * kTmaStages + 2 * kTmaStages * 8;
}

// Consumer side of a staged chunk: the lane's words of slice `warp`, with the
// unaligned tail (V * sizeof(T) not a multiple of 16) from global and padding
// after V.
template <typename T>
__device__ __forceinline__ void stage_slice(const T* st, const T* grow, int n_el, int c0,
                                            uint4 (&r)[Traits<T>::NV]) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, CH = chunk_elems<T>(), SL = sub_elems<T>();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (n_el == CH) {
#pragma unroll
    for (int v = 0; v < NV; ++v) r[v] = *reinterpret_cast<const uint4*>(st + warp * SL + (v * 32 + lane) * VEC);
    return;
  }
  const int bulk_el = (int)(((uint32_t)(n_el * (int)sizeof(T)) & ~15u) / sizeof(T));
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int e0 = warp * SL + (v * 32 + lane) * VEC;
    T b[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const int idx = e0 + e;
      b[e] = idx < bulk_el ? st[idx] : idx < n_el ? grow[c0 + idx] : pad_bits<T>();
    }
    r[v] = *reinterpret_cast<const uint4*>(b);
  }
}

template <typename T>
__global__ void __launch_bounds__(kTmaThreads, kTmaCtas) k_stream_tma(StreamArgs a) {
  constexpr int CH = chunk_elems<T>(), ROWB = stage_row_bytes<T>(), NV = Traits<T>::NV;
  extern __shared__ __align__(128) uint8_t smem[];
  int4* sdesc = reinterpret_cast<int4*>(smem + kTmaStages * 2 * ROWB);  // (trow lo, trow hi, c, -)
  uint64_t* full = reinterpret_cast<uint64_t*>(sdesc + kTmaStages);
  uint64_t* consumed = full + kTmaStages;
  const int nc = a.nsub / kCWarps;
  const long long n_items = (long long)stream_rows(a) * nc;
  const int G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&consumed[s], kCWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCWarps) {
    // ---------------- TMA producer (whole warp tracks the row cursor) ----------------
    int seq = 0, s = 0;
    uint32_t round = 0;
    for (long long q = blockIdx.x; q < n_items; q += G) {
      const long long r = q / nc;
      const int c = (int)(q - r * nc);
      seq = seq_of_row(a.cu_sl, a.B, seq, r);
      if (round > 0) mbar_wait(&consumed[s], (round - 1) & 1u);
      if (lane == 0) {
        const long long trow = r + seq;
        sdesc[s] = make_int4((int)(trow & 0xffffffff), (int)(trow >> 32), c, 0);
        const int c0 = c * CH;
        const int n_el = min(CH, a.V - c0);
        const uint32_t bytes = n_el > 0 ? (uint32_t)(n_el * (int)sizeof(T)) & ~15u : 0u;
        uint8_t* dst = smem + s * 2 * ROWB;
        if (bytes) {
          mbar_arrive_expect_tx(&full[s], 2 * bytes);
          bulk_g2s(dst, reinterpret_cast<const T*>(a.tl) + trow * a.ld_t + c0, bytes, &full[s]);
          bulk_g2s(dst + ROWB, reinterpret_cast<const T*>(a.dl) + r * a.ld_d + c0, bytes, &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      if (++s == kTmaStages) {
        s = 0;
        ++round;
      }
    }
    return;
  }

  // ---------------- consumer warps ----------------
  int s = 0;
  uint32_t round = 0;
  for (long long q = blockIdx.x; q < n_items; q += G) {
    const long long r = q / nc;
    mbar_wait(&full[s], round & 1u);
    const int4 dsc = sdesc[s];
    const int c = dsc.z;
    const long long trow = (long long)(uint32_t)dsc.x | ((long long)dsc.y << 32);
    const int c0 = c * CH;
    const int n_el = max(0, min(CH, a.V - c0));
    const T* st = reinterpret_cast<const T*>(smem + s * 2 * ROWB);
    uint4 rt[NV], rd[NV];
    stage_slice<T>(st, reinterpret_cast<const T*>(a.tl) + trow * a.ld_t, n_el, c0, rt);
    stage_slice<T>(st + CH, reinterpret_cast<const T*>(a.dl) + r * a.ld_d, n_el, c0, rd);
    __syncwarp();
    if (lane == 0) mbar_arrive(&consumed[s]);
    if (++s == kTmaStages) {
      s = 0;
      ++round;
    }
    store_partial(a.part + r * a.nsub + c * kCWarps + warp, slice_stats<T>(rt, rd));
  }
}

#include "verify_draw.cuh"   // a2-a4 kernels (inside namespace dsde)
#include "verify_fused.cuh"  // the whole step in one persistent kernel

// 0 = stream kernel + k_tail (default), 1 = stream kernel + split finalize /
// draw / select, 2 = one persistent kernel k_fused (DSDE_TAIL=tail|split|fused)
static int tail_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DSDE_TAIL");
    v = !e ? 0 : strcmp(e, "split") == 0 ? 1 : strcmp(e, "fused") == 0 ? 2 : 0;
  }
  return v;
}

// k_tail CTA shape: 16 warps while B <= this many sequences per SM, else 8
#ifndef DSDE_TAIL16_MAXB_PER_SM
#define DSDE_TAIL16_MAXB_PER_SM 2
#endif
// 32-warp CTAs (one per SM) while B <= this many sequences per SM (0 = never)
#ifndef DSDE_TAIL32_MAXB_PER_SM
#define DSDE_TAIL32_MAXB_PER_SM 1
#endif

// Launch with programmatic stream serialization (PDL): the kernel may start
// while the previous kernel on the stream drains and must call
// griddepcontrol.wait before touching that kernel's results. DSDE_PDL=0
// launches it plainly (griddepcontrol.wait is then a no-op).
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
  static int use = -1;
  if (use < 0) {
    const char* e = getenv("DSDE_PDL");
    use = (e && strcmp(e, "0") == 0) ? 0 : 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

static int stream_variant() {  // 0 = ldg (default), 1 = tma (DSDE_STREAM=tma)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DSDE_STREAM");
    v = (e && strcmp(e, "tma") == 0) ? 1 : 0;
  }
  return v;
}

template <typename KernelT>
static int resident_grid(KernelT k, int threads, int smem, int sms, int cap_per_sm) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem);
  per_sm = std::max(1, cap_per_sm > 0 ? std::min(per_sm, cap_per_sm) : per_sm);
  return per_sm * sms;
}

// step != nullptr: the whole-step launch (dsde_step) with the signal (and, if
// step->fuse_cap, the cap) fused into the tail kernel.
template <typename T>
cudaError_t launch_verify(int B, int V, int total, const int32_t* cu_sl, const int32_t* tokens,
                          const void* tl, int64_t ld_t, const void* dl, int64_t ld_d,
                          const uint64_t* seeds, int32_t* acc_len, int32_t* emitted, float* kld,
                          uint8_t* flags, const VerifyWs& ws, int32_t* err, Profiler* prof,
                          cudaStream_t s, const StepExtra* step = nullptr, int greedy = 0,
                          int dev_rows = 0, float* ent = nullptr) {
  const bool pr = prof != nullptr && prof->on;
  auto mark = [&]() {
    if (pr) cudaEventRecord(prof->next(), s);
  };
  const int ns = n_subs(V, sizeof(T) == 2 ? DSDE_BF16 : DSDE_F32, stream_variant() == 1);
  int dev = 0;
  cudaGetDevice(&dev);
  struct Grids {
    int sms = 0, ldg = 0, ldg_ent = 0, tma = 0, draw = 0;
  };
  static Grids grids[64];
  Grids& g = grids[dev & 63];
  if (g.sms == 0) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(k_stream_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, tma_smem<T>());
    g.ldg = resident_grid(k_stream_ldg<T, false>, kLdgThreads, 0, sms, 0);
    g.ldg_ent = resident_grid(k_stream_ldg<T, false, true>, kLdgThreads, 0, sms, 0);
    g.tma = resident_grid(k_stream_tma<T>, kTmaThreads, tma_smem<T>(), sms, kTmaCtas);
    g.draw = resident_grid(k_draw_ldg<T>, kLdgThreads, 0, sms, 0);
    g.sms = sms;
  }
  const int variant = ent ? 0 : stream_variant();  // the draft entropy is in the ldg kernel only
  // the fused kernel has no T = 0 mode and sizes its counters from the host total
  const int tv = (greedy || dev_rows || ent) && tail_variant() == 2 ? 0 : tail_variant();
  if (tv == 2) {
    static int fused_grid[64] = {0};
    int& fg = fused_grid[dev & 63];
    if (fg == 0) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused<T>, kFusedThreads, 0);
      fg = std::max(1, per_sm) * g.sms;
    }
    mark();
    FusedArgs fa2{};
    fa2.B = B;
    fa2.V = V;
    fa2.total = total;
    fa2.nsub = ns;
    fa2.nd = n_subs_d(V, sizeof(T) == 2 ? DSDE_BF16 : DSDE_F32);
    fa2.cu_sl = cu_sl;
    fa2.tokens = tokens;
    fa2.tl = tl;
    fa2.ld_t = ld_t;
    fa2.dl = dl;
    fa2.ld_d = ld_d;
    fa2.seeds = seeds;
    fa2.part = ws.part;
    fa2.rowres = reinterpret_cast<RowRes*>(ws.rowres);
    fa2.rec = ws.rec;
    fa2.smass = ws.mass;
    fa2.sref = ws.ref;
    fa2.acc_len = acc_len;
    fa2.emitted = emitted;
    fa2.kld = kld;
    fa2.flags = flags;
    fa2.err = err;
    fa2.ctl = reinterpret_cast<FusedCtl*>(ws.counters);
    fa2.row_cnt = ws.counters + kCtlInts;
    fa2.seq_cnt = fa2.row_cnt + total;
    fa2.draw_cnt = fa2.seq_cnt + B;
    fa2.fin = fa2.draw_cnt + B;
    fa2.queue = fa2.fin + B;
    fa2.step = step != nullptr;
    fa2.fuse_cap = step != nullptr && step->fuse_cap;
    if (step) {
      fa2.sig = step->sig;
      fa2.cap = step->cap;
    }
    cudaError_t e = cudaMemsetAsync(ws.counters, 0, ws.counter_bytes, s);
    if (e != cudaSuccess) return e;
    const long long units = (long long)total * ns;
    const int grid = (int)std::min<long long>(fg, std::max<long long>(1, (units + 7) / 8));
    // a plain launch: stream units are claimed dynamically and every wait is on
    // a sequence whose rows resident warps produce, so co-residency of the
    // whole grid is not required (a cooperative launch measured ~2x slower)
    k_fused<T><<<grid, kFusedThreads, 0, s>>>(fa2);
    mark();
    mark();
    mark();
    mark();
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  mark();
  // a1: statistics of every (draft row, vocab slice)
  StreamArgs sa{tl, ld_t, dl, ld_d, cu_sl, B, V, ns, total, ws.part, dev_rows};
  if (variant == 1) {
    const long long items = (long long)total * (ns / kCWarps);
    k_stream_tma<T><<<(int)std::min<long long>(items, g.tma), kTmaThreads, tma_smem<T>(), s>>>(sa);
  } else {
    const long long units = (long long)total * ns;
    const long long blocks = (units + kLdgThreads / 32 - 1) / (kLdgThreads / 32);
    const int grid = (int)std::min<long long>(blocks, ent ? g.ldg_ent : g.ldg);
    if (ent) {
      if (dev_rows) k_stream_ldg<T, true, true><<<grid, kLdgThreads, 0, s>>>(sa);
      else k_stream_ldg<T, false, true><<<grid, kLdgThreads, 0, s>>>(sa);
    } else {
      if (dev_rows) k_stream_ldg<T, true><<<grid, kLdgThreads, 0, s>>>(sa);
      else k_stream_ldg<T, false><<<grid, kLdgThreads, 0, s>>>(sa);
    }
  }
  mark();
  // a2-a3: row merge, KL, accept test, layout, draw record
  FinArgs fa{B, V, total, ns, cu_sl, tokens, tl, ld_t, dl, ld_d, seeds, ws.part,
             acc_len, emitted, kld, flags, ws.rec, err, greedy, dev_rows, ent};
  const int nd = n_subs_d(V, sizeof(T) == 2 ? DSDE_BF16 : DSDE_F32);
  DrawArgs da{B, V, nd, tl, ld_t, dl, ld_d, ws.rec, ws.mass, ws.ref};
  SelArgs sel{B, V, nd, tl, ld_t, dl, ld_d, ws.rec, ws.mass, ws.ref, emitted, flags, err};
  if (step) {
    // 16-warp CTAs while every sequence gets a resident CTA (2 per SM), 8-warp
    // CTAs (4 per SM) for larger batches so the tail stays one wave longer
    if (B <= DSDE_TAIL32_MAXB_PER_SM * g.sms)
      launch_pdl(k_tail<T, true, 32>, B, 1024, s, fa, da, sel, *step);
    else if (B <= DSDE_TAIL16_MAXB_PER_SM * g.sms)
      launch_pdl(k_tail<T, true, 16>, B, 512, s, fa, da, sel, *step);
    else
      launch_pdl(k_tail<T, true, 8>, B, 256, s, fa, da, sel, *step);
    mark();
    mark();
    mark();
    return cudaGetLastError();
  }
  if (tv == 0) {
    // a2-a4 fused: one CTA per sequence (the profiler's later phases read 0)
    if (B <= DSDE_TAIL32_MAXB_PER_SM * g.sms)
      launch_pdl(k_tail<T, false, 32>, B, 1024, s, fa, da, sel, StepExtra{});
    else if (B <= DSDE_TAIL16_MAXB_PER_SM * g.sms)
      launch_pdl(k_tail<T, false, 16>, B, 512, s, fa, da, sel, StepExtra{});
    else
      launch_pdl(k_tail<T, false, 8>, B, 256, s, fa, da, sel, StepExtra{});
    mark();
    mark();
    mark();
    return cudaGetLastError();
  }
  k_finalize<T><<<B, kFinThreads, 0, s>>>(fa);
  mark();
  // a4: draw-weight masses of the drawn rows, then the inverse-CDF select
  {
    const long long units = (long long)B * nd;
    const long long blocks = (units + kLdgThreads / 32 - 1) / (kLdgThreads / 32);
    k_draw_ldg<T><<<(int)std::min<long long>(blocks, g.draw), kLdgThreads, 0, s>>>(da);
  }
  mark();
  k_select<T><<<(B + 3) / 4, 128, 0, s>>>(sel);
  mark();
  return cudaGetLastError();
}

}  // namespace dsde

using namespace dsde;

extern "C" size_t dsde_verify_workspace_size(int B, int total_draft_rows, int V, dsde_dtype dtype) {
  if (B < 1 || V < 2 || total_draft_rows < 0) return 0;
  if (dtype != DSDE_F32 && dtype != DSDE_BF16) return 0;
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
  if ((long long)(total_draft_rows + B) * n_subs(V, dtype) > 0x7fffffffLL) return DSDE_ERR_ARG;
  VerifyWs ws;
  ws_layout(B, total_draft_rows, V, dtype, &ws, reinterpret_cast<char*>(workspace));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (dtype == DSDE_BF16)
    e = launch_verify<uint16_t>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                                draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld,
                                flags, ws, st->err, st->prof, s, nullptr, st->cfg.greedy, st->cfg.device_rows,
                                st->entropy_out);
  else
    e = launch_verify<float>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                             draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld, flags,
                             ws, st->err, st->prof, s, nullptr, st->cfg.greedy, st->cfg.device_rows,
                                st->entropy_out);
  return e == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

// Implemented in api.cu / signal.cu.
dsde_status dsde_comm_allreduce_i64(dsde_comm comm, long long* buf, int n_sum, int max_at,
                                    cudaStream_t s);
namespace dsde {
cudaError_t launch_cap_multi(const CapArgs& a, dsde_comm comm, cudaStream_t s, dsde_status* st);
}

extern "C" dsde_status dsde_step(dsde_state st, int B, int V, dsde_dtype dtype, int total_draft_rows,
                                 const int32_t* slots, const int32_t* cu_sl,
                                 const int32_t* draft_tokens, const void* target_logits,
                                 int64_t ld_t, const void* draft_logits, int64_t ld_d,
                                 const uint64_t* seeds, const int32_t* budget,
                                 int32_t* accepted_len, int32_t* emitted_tokens, float* kld,
                                 uint8_t* flags, int32_t* sl_hat, double* diag, int32_t* next_sl,
                                 int32_t* cap, void* workspace, size_t ws_bytes, dsde_comm comm,
                                 void* stream) {
  if (!st || !slots || !sl_hat || !next_sl || !cap || !cu_sl || !draft_tokens || !target_logits ||
      !draft_logits || !seeds || !accepted_len || !emitted_tokens || !kld || !workspace)
    return DSDE_ERR_ARG;
  if (B < 1 || V < 2 || total_draft_rows < B || total_draft_rows > B * DSDE_MAX_SL)
    return DSDE_ERR_ARG;
  if (B > st->max_seqs) return DSDE_ERR_STATE;
  if (dtype != DSDE_F32 && dtype != DSDE_BF16) return DSDE_ERR_ARG;
  if (ld_t < V || ld_d < V) return DSDE_ERR_ARG;
  const size_t esz = dtype == DSDE_BF16 ? 2 : 4;
  if ((((uintptr_t)target_logits) | ((uintptr_t)draft_logits)) & 15) return DSDE_ERR_ARG;
  if (((size_t)ld_t * esz) % 16 || ((size_t)ld_d * esz) % 16) return DSDE_ERR_ARG;
  if (((uintptr_t)workspace) & 255) return DSDE_ERR_ARG;
  if (ws_bytes < ws_layout(B, total_draft_rows, V, dtype, nullptr, nullptr)) return DSDE_ERR_ARG;
  if ((long long)(total_draft_rows + B) * n_subs(V, dtype) > 0x7fffffffLL) return DSDE_ERR_ARG;
  VerifyWs ws;
  ws_layout(B, total_draft_rows, V, dtype, &ws, reinterpret_cast<char*>(workspace));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  StepExtra x;
  x.sig = SignalArgs{st->cfg, B, st->max_seqs, slots, cu_sl, kld, accepted_len, sl_hat, diag,
                     st->seq, st->err};
  x.cap = CapArgs{st->cfg, B, st->max_seqs, slots, sl_hat, budget, next_sl, cap, st->seq, st->scratch};
  x.fuse_cap = comm == nullptr;
  x.counter = reinterpret_cast<unsigned*>(st->scratch + 4);
  cudaError_t e;
  if (dtype == DSDE_BF16)
    e = launch_verify<uint16_t>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                                draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld,
                                flags, ws, st->err, st->prof, s, &x, st->cfg.greedy, st->cfg.device_rows,
                                st->entropy_out);
  else
    e = launch_verify<float>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                             draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld, flags,
                             ws, st->err, st->prof, s, &x, st->cfg.greedy, st->cfg.device_rows,
                                st->entropy_out);
  if (e != cudaSuccess) return DSDE_ERR_CUDA;
  if (!comm) return DSDE_OK;
  dsde_status rs = DSDE_OK;
  e = launch_cap_multi(x.cap, comm, s, &rs);
  if (rs != DSDE_OK) return rs;
  return e == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

#if DSDE_TAIL_TRACE
// measurement build only: copy n CTA records (6 u64 each: after the PDL wait,
// after finalize, after the draw, after the select, -, smid << 8 | mode)
extern "C" int dsde_debug_tail_trace(unsigned long long* host, int n) {
  n = n < dsde::kTraceMax ? n : dsde::kTraceMax;
  return cudaMemcpyFromSymbol(host, dsde::g_tail_trace, sizeof(unsigned long long) * 6 * n) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" dsde_status dsde_set_draft_entropy(dsde_state st, float* entropy) {
  if (!st) return DSDE_ERR_ARG;
  st->entropy_out = entropy;
  return DSDE_OK;
}

