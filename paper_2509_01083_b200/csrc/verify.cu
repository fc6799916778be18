// verify.cu — dsde_verify / dsde_step: the speculative-verification pass
// (§8(a) a1-a4; with dsde_step also a5-a7).
//
// Launch sequence (on the caller's stream, no host synchronisation):
//   1. k_stream_ldg: persistent warps stream every (draft position row, vocab
//      slice) of the target and draft logits once (a1: per 2048-token bf16 /
//      512-token fp32 slice S = sum e_v, A = sum e_v w_v, D = sum e_v g(w_v)
//      about the slice reference) and write 32-byte slice partials;
//   2. k_tail (tail.cuh), launched with programmatic dependent launch: one CTA
//      per sequence merges its rows in fp64 (KL, log p/q, Philox accept test,
//      a2), lays it out (a3), draws its token (a4: D7 inverse CDF over the drawn
//      row, or the D23 proposals from p for a recovery draw) and, in dsde_step, updates
//      its signal and SL^ (a5-a6); the last signal applies the batch cap (a7,
//      single GPU);
//   3. (dsde_step with a communicator) k_cap_partial, ncclAllReduce, k_cap_apply.
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
template <>
struct Traits<uint16_t> {                  // bf16 bit patterns
  static constexpr int VEC = 8;            // elements per 16-byte vector
  static constexpr int NV = DSDE_NV_BF16;  // vectors per lane per stream slice (2048 tokens)
  static constexpr int NVD = 4;            // vectors per lane per draw slice (1024 tokens)
};
template <>
struct Traits<float> {
  static constexpr int VEC = 4;
  static constexpr int NV = 4;   // 512 tokens
  static constexpr int NVD = 4;  // 512 tokens
};
// one warp's slice of a row: 32 lanes x NV vectors x VEC elements
template <typename T>
__host__ __device__ constexpr int sub_elems() {
  return 32 * Traits<T>::VEC * Traits<T>::NV;
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
  float M;           // reference max of t / T (residual)
  float invT;        // 1 / T of the sequence (D20; 1 for greedy)
  double C;          // reference t - d (residual)
  double lam;        // log1p(y) = log(sum_v p_v exp(-w_v)) (residual)
  double u;          // u_smp of the slot
  double S;          // sum_v exp(t_v - M) of the drawn row (residual)
};
static_assert(sizeof(SeqRec) == 64, "SeqRec layout");

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// one warp's slice of a row in the draw and select passes
template <typename T>
__host__ __device__ constexpr int draw_elems() {
  return 32 * Traits<T>::VEC * Traits<T>::NVD;
}

// stream slices per row (2048 tokens bf16, 512 fp32)
inline int n_subs(int V, dsde_dtype dt) {
  const int se = dt == DSDE_BF16 ? sub_elems<uint16_t>() : sub_elems<float>();
  return (V + se - 1) / se;
}
// draw slices per row (1024 tokens bf16, 512 fp32)
inline int n_draws(int V, dsde_dtype dt) {
  const int se = dt == DSDE_BF16 ? draw_elems<uint16_t>() : draw_elems<float>();
  return (V + se - 1) / se;
}

// Workspace of dsde_verify / dsde_step (caller-owned, 256-byte aligned): the
// slice partials (32 B per draft row x slice: 1.6% of the logit bytes),
// per-sequence draw records (64 B), per-slice draw masses (12 B per slice of
// each sequence's drawn row) and the tail's signal counter.
struct VerifyWs {
  void* part;   // SubPartial [total * nsub]
  void* rec;    // SeqRec [B]
  double* mass;  // [B * nsub]
  float* mref;   // [B * nsub]
  int* counters;  // [8]: [0] signals done (zeroed by the stream kernel)
  size_t counter_bytes;
};

inline size_t ws_layout(int B, int total, int V, dsde_dtype dt, VerifyWs* ws, char* base) {
  const int ns = n_subs(V, dt), nd = n_draws(V, dt);
  const size_t p_bytes = align256((size_t)32 * total * ns);
  const size_t r_bytes = align256((size_t)64 * B);
  const size_t m_bytes = align256(sizeof(double) * (size_t)B * nd);
  const size_t x_bytes = align256(sizeof(float) * (size_t)B * nd);
  const size_t cnt = 8;
  const size_t c_bytes = align256(sizeof(int) * cnt);
  if (ws) {
    size_t o = 0;
    ws->part = base + o;
    o += p_bytes;
    ws->rec = base + o;
    o += r_bytes;
    ws->mass = reinterpret_cast<double*>(base + o);
    o += m_bytes;
    ws->mref = reinterpret_cast<float*>(base + o);
    o += x_bytes;
    ws->counters = reinterpret_cast<int*>(base + o);
    ws->counter_bytes = sizeof(int) * cnt;
  }
  return p_bytes + r_bytes + m_bytes + x_bytes + c_bytes;
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

// w = (t - d) / T - C with the difference t - d exact (bf16) or carried as
// hi + lo (fp32, TwoDiff) and one rounding for the scale and the reference;
// invT = 1 gives exactly the FADD of (t - d) and -C.
template <typename T>
__device__ __forceinline__ float2 diff2(float2 t, float2 d, float C, float invT);
template <>
__device__ __forceinline__ float2 diff2<uint16_t>(float2 t, float2 d, float C, float invT) {
  return __ffma2_rn(__fadd2_rn(t, make_float2(-d.x, -d.y)), make_float2(invT, invT), make_float2(-C, -C));
}
template <>
__device__ __forceinline__ float2 diff2<float>(float2 t, float2 d, float C, float invT) {
  // (an infinite difference — a masked logit, D21 — keeps its sign: lo = 0)
  float2 r;
  {
    const float hi = __fsub_rn(t.x, d.x), bb = __fsub_rn(hi, t.x);
    float lo = __fadd_rn(__fsub_rn(t.x, __fsub_rn(hi, bb)), __fsub_rn(-d.x, bb));
    if (!(fabsf(hi) < INFINITY)) lo = 0.f;
    r.x = __fadd_rn(__fmaf_rn(hi, invT, -C), __fmul_rn(lo, invT));
  }
  {
    const float hi = __fsub_rn(t.y, d.y), bb = __fsub_rn(hi, t.y);
    float lo = __fadd_rn(__fsub_rn(t.y, __fsub_rn(hi, bb)), __fsub_rn(-d.y, bb));
    if (!(fabsf(hi) < INFINITY)) lo = 0.f;
    r.y = __fadd_rn(__fmaf_rn(hi, invT, -C), __fmul_rn(lo, invT));
  }
  return r;
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

// Per-slice constants of the a1 sums about the reference (M, C = M - max d),
// at temperature T (D20): logits enter as t / T, so the reference is the raw
// maxima times invT = 1/T and the exponent scale is invT log2 e (both exact
// copies of the untempered constants when invT = 1).
struct SumRef {
  float2 nML2, nDL2, L2s;
  float Cw, invT;
  __device__ __forceinline__ SumRef(float M, float Dmax, float inv_t = 1.f) {
    invT = inv_t;
    const float Ms = M * inv_t, Ds = Dmax * inv_t;
    Cw = Ms - Ds;
    const float ML2 = Ms * kLog2e, DL2 = Ds * kLog2e, l2 = kLog2e * inv_t;
    nML2 = make_float2(-ML2, -ML2);
    nDL2 = make_float2(-DL2, -DL2);
    L2s = make_float2(l2, l2);
  }
};

// Masked-logit sums (D21; dsde_config.masked): Fp = sum of e e^{-w} (the
// draft mass on supp p, in e's frame: p's reference minus C), Fm = sum of
// e^{d/T - max d/T} over the tokens the target masks (draft mass outside
// supp p, about the slice's max d); cc = some token the draft masks has p > 0
// (then KL(p||q) = +inf).
struct MaskAcc {
  float2 Fp, Fm;
  int cc;
};

// a1 accumulation of one element pair (packed FFMA2 math, two MUFU.EX2 per
// element): S += e, A += e w, D += e g(w).
// ENT (opt-in): also Sd += f and E += f (d - max d), f = e^{d - max d},
// the draft's own softmax sums about the slice max of d (H(q) = log Sd - E / Sd).
struct EntAcc {
  float2 Sd, E;
};

template <typename T, bool ENT = false, bool MASK = false>
__device__ __forceinline__ void pair_accum_w(float2 tt, float2 dd, float2 w, const SumRef& R, float2& S2,
                                             float2& A2, float2& D2, EntAcc* ent = nullptr,
                                             MaskAcc* mk = nullptr) {
  const float2 L2 = R.L2s;
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
  const float2 e = make_float2(fast_exp2(xt.x), fast_exp2(xt.y));
  if constexpr (MASK) {
    // t = -inf (p_v = 0): e = 0, the draft mass e^{d/T - max d/T} goes to Fm;
    // d = -inf while t is finite (q_v = 0 < p_v): KL = +inf (cc); either way w
    // is replaced by 0 so that A and D get exact zeros instead of 0 * inf
    const bool mtx = tt.x == -INFINITY, mty = tt.y == -INFINITY;
    const bool mdx = dd.x == -INFINITY, mdy = dd.y == -INFINITY;
    const float2 arg = __ffma2_rn(dd, L2, R.nDL2);
    mk->Fm = __fadd2_rn(mk->Fm, make_float2(mtx ? fast_exp2(arg.x) : 0.f, mty ? fast_exp2(arg.y) : 0.f));
    mk->cc |= (mdx && !mtx) || (mdy && !mty);
    w = make_float2((mtx || mdx) ? 0.f : w.x, (mty || mdy) ? 0.f : w.y);
  }
  // f = e e^{-w} = e^{d/T - (M/T - C)}, formed from e's own exponent so that
  // e, f and w share one reference (a separately rounded reference for f would
  // shift f against e by the rounding of (max d / T) log2 e, which the
  // cancellation in f - e + e w amplifies); the exponent is <= 0 up to the
  // slice reference, so f never overflows for finite inputs
  const float2 xf = __ffma2_rn(w, make_float2(-kLog2e, -kLog2e), xt);
  float2 f = make_float2(fast_exp2(xf.x), fast_exp2(xf.y));
  if constexpr (MASK) {
    if (dd.x == -INFINITY) f.x = 0.f;  // q_v = 0
    if (dd.y == -INFINITY) f.y = 0.f;
    mk->Fp = __fadd2_rn(mk->Fp, f);
  }
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
  // (masked elements have w = 0: the polynomial branch, exactly 0)
  const float2 term = make_float2(fabsf(w.x) < 1.f ? sm.x : bg.x, fabsf(w.y) < 1.f ? sm.y : bg.y);
  D2 = __fadd2_rn(D2, term);
  if constexpr (ENT) {
    // the draft's own sums in the same frame: Sd = sum f, E = sum f ln f
    ent->Sd = __fadd2_rn(ent->Sd, f);
    ent->E = __ffma2_rn(f, __fmul2_rn(xf, make_float2(kLn2, kLn2)), ent->E);
  }
}

template <typename T, bool ENT = false, bool MASK = false>
__device__ __forceinline__ void pair_accum(float2 tt, float2 dd, const SumRef& R, float2& S2, float2& A2,
                                           float2& D2, EntAcc* ent = nullptr, MaskAcc* mk = nullptr) {
  pair_accum_w<T, ENT, MASK>(tt, dd, diff2<T>(tt, dd, R.Cw, R.invT), R, S2, A2, D2, ent, mk);
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
template <typename T, bool ENT = false, bool MASK = false>
__device__ __forceinline__ void vec_accum(const uint4& t, const uint4& d, const SumRef& R, float2& S2,
                                          float2& A2, float2& D2, EntAcc* ent = nullptr, MaskAcc* mk = nullptr) {
  constexpr int P = Traits<T>::VEC / 2;
  const uint4 rt[1] = {t}, rd[1] = {d};
  if constexpr (MASK) {
    // masked logits (D21): every element takes the exact per-element path,
    // which handles the -inf cases
#pragma unroll
    for (int h = 0; h < Traits<T>::VEC; h += 2)
      pair_accum<T, false, true>(pair_of<T>(rt, h), pair_of<T>(rd, h), R, S2, A2, D2, nullptr, mk);
    return;
  }
#if DSDE_WIDE_POLY
  float2 tt[P], w[P];
  float am = 0.f;
#pragma unroll
  for (int h = 0; h < P; ++h) {
    tt[h] = pair_of<T>(rt, 2 * h);
    w[h] = diff2<T>(tt[h], pair_of<T>(rd, 2 * h), R.Cw, R.invT);
    am = fmaxf(am, fmaxf(fabsf(w[h].x), fabsf(w[h].y)));
  }
  constexpr float kWideR = 2.f;
  if (__all_sync(kFull, am < kWideR)) {
    const float2 L2 = R.L2s;
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
        // f = e e^{-w} = e (1 - w + w^2 h(-w)); ln f = xt ln 2 - w (the frame of
        // the exact path)
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

// The warp's three sums by recursive halving (6 shuffles instead of 15):
// after the xor-16 and xor-8 rounds lanes 0-7 hold partial S, 8-15 A, 16-23 D;
// three more rounds complete them; lane 0 gathers A and D.
__device__ __forceinline__ SubPartial finish_partial(float2 S2, float2 A2, float2 D2, float M, float Dmax,
                                                     float Cw) {
  const int lane = threadIdx.x & 31;
  float s = S2.x + S2.y, aa = A2.x + A2.y;
  const float dd = D2.x + D2.y;
  {  // xor 16: lanes < 16 keep (S, A), lanes >= 16 keep (D, 0)
    const bool up = lane & 16;
    const float k0 = up ? dd : s, k1 = up ? 0.f : aa;
    const float s0 = up ? s : dd, s1 = up ? aa : 0.f;
    s = k0 + __shfl_xor_sync(kFull, s0, 16);
    aa = k1 + __shfl_xor_sync(kFull, s1, 16);
  }
  {  // xor 8: lanes with bit 3 clear keep the first, set keep the second
    const bool up = lane & 8;
    const float k0 = up ? aa : s, s0 = up ? s : aa;
    s = k0 + __shfl_xor_sync(kFull, s0, 8);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
  SubPartial p;
  p.pad0 = p.pad1 = 0.f;
  p.S = s;
  p.A = __shfl_sync(kFull, s, 8);
  p.D = __shfl_sync(kFull, s, 16);
  p.M = M;
  p.C = Cw;
  p.maxd = Dmax;
  return p;
}

// `after_max` runs (warp-uniformly) once the slice maxima are reduced over the
// warp, i.e. once every lane's words have been consumed. invT = 1/T of the
// row's sequence (D20). MASK (D21): the partial's spare words carry Fm (its sign bit:
// cc) and Fp
// (MaskAcc); a slice whose target logits are all masked keeps its draft mass
// (reference max d, M = -inf in the partial).
template <typename T, int NV, typename Hook = NoHook, bool ENT = false, bool MASK = false>
__device__ __forceinline__ SubPartial slice_stats(const uint4 (&rt)[NV], const uint4 (&rd)[NV], float invT = 1.f,
                                                  Hook after_max = Hook()) {
  LaneMax<T> mx;
  mx.init();
#pragma unroll
  for (int v = 0; v < NV; ++v) mx.add(rt[v], rd[v]);
  float M, Dmax;
  mx.reduce(M, Dmax);
  after_max();
  bool t_masked = false;
  if constexpr (MASK) {
    // every t masked (or row padding), some d kept: keep the draft mass with a
    // finite reference (all e = 0); every d masked, some t kept: a finite
    // draft reference (C = 0; every kept t is then a KL = +inf token)
    t_masked = M <= -1e30f && Dmax > -1e30f;
    if (t_masked) M = Dmax;
    if (Dmax <= -1e30f && M > -1e30f) Dmax = M;
  }
  if (M <= -1e30f) return empty_partial();  // slice beyond V (padding only; NaN is not empty)
  const SumRef R(M, Dmax, invT);
  float2 S2 = make_float2(0.f, 0.f), A2 = S2, D2 = S2;
  if constexpr (ENT) {
    EntAcc ent{S2, S2};
#pragma unroll
    for (int v = 0; v < NV; ++v) vec_accum<T, true>(rt[v], rd[v], R, S2, A2, D2, &ent);
    SubPartial p = finish_partial(S2, A2, D2, M * invT, Dmax * invT, R.Cw);
    float Sd = ent.Sd.x + ent.Sd.y, E = ent.E.x + ent.E.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Sd += __shfl_xor_sync(kFull, Sd, o);
      E += __shfl_xor_sync(kFull, E, o);
    }
    p.pad0 = Sd;
    p.pad1 = E;
    return p;
  } else if constexpr (MASK) {
    MaskAcc mk{S2, S2, 0};
#pragma unroll
    for (int v = 0; v < NV; ++v) vec_accum<T, false, true>(rt[v], rd[v], R, S2, A2, D2, nullptr, &mk);
    SubPartial p = finish_partial(S2, A2, D2, M * invT, Dmax * invT, R.Cw);
    float Fp = mk.Fp.x + mk.Fp.y, Fm = mk.Fm.x + mk.Fm.y;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Fp += __shfl_xor_sync(kFull, Fp, o);
      Fm += __shfl_xor_sync(kFull, Fm, o);
    }
    const int cc = __any_sync(kFull, mk.cc);
    p.pad0 = __int_as_float(__float_as_int(Fm) | (cc ? (int)0x80000000u : 0));  // sign bit: cc
    p.pad1 = Fp;
    if (t_masked) {
      p.M = -INFINITY;
      p.C = 0.f;
    }
    return p;
  } else {
#pragma unroll
    for (int v = 0; v < NV; ++v) vec_accum<T>(rt[v], rd[v], R, S2, A2, D2);
    return finish_partial(S2, A2, D2, M * invT, Dmax * invT, R.Cw);
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
  int* ctl;               // the tail's signal counter, zeroed here (the tail reads it after griddepcontrol.wait)
  const float* temps;     // [B] per-sequence temperature (dsde_set_temperature, D20) or NULL
};

// 1/T of sequence i (D20): T > 0 samples at T; T = 0 (greedy) and a missing or
// invalid temperature use the stored logits (T = 1; the finalize reports an
// invalid one)
__device__ __forceinline__ float inv_temp(const float* temps, int i) {
  if (!temps) return 1.f;
  const float T = __ldg(temps + i);
  return (T > 0.f && T < INFINITY) ? 1.f / T : 1.f;
}

// rows this launch streams: the host's Σk_i, or (device_rows) cu_sl[B] clamped
// to the capacity the grid and workspace were sized for
__device__ __forceinline__ int stream_rows(const StreamArgs& a) {
  return a.dev_rows ? min(max(__ldg(a.cu_sl + a.B), 0), a.total) : a.total;
}

// ---------------------------------------------------------------------------
// a1: persistent warps over the units q = (draft row r, slice u), q = global
// warp + j * (total warps), row-major so rows complete in order. Per unit each
// lane issues its NV + NV 16-byte non-allocating loads at once (the whole
// 2048-token slice pair of the warp), reduces the slice maxima (the reference)
// and accumulates S, A, D; no shared memory, no block barriers.
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
template <typename T, bool DEV_ROWS, bool ENT = false, bool MASK = false>
__global__ void __launch_bounds__(kLdgThreads, (ENT || MASK) ? DSDE_ENT_MINB : DSDE_LDG_MINB) k_stream_ldg(StreamArgs a) {
  constexpr int NV = Traits<T>::NV;
  const int total = DEV_ROWS ? stream_rows(a) : a.total;
  const long long n_units = (long long)total * a.nsub;
  const long long W = (long long)gridDim.x * (kLdgThreads / 32);
  long long q = (long long)blockIdx.x * (kLdgThreads / 32) + (threadIdx.x >> 5);
  if (q == 0 && a.ctl) *a.ctl = 0;
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
    store_partial(dst, slice_stats<T, NV, NoHook, ENT, MASK>(rt, rd, inv_temp(a.temps, seq)));
#endif
    u += du;
    r += dr;
    if (u >= a.nsub) {
      u -= a.nsub;
      ++r;
    }
  }
}

#include "verify_draw.cuh"  // a2-a4 device functions (inside namespace dsde)
struct StepExtra {  // the whole-step launch (dsde_step): signal (a5-a6) and cap (a7)
  SignalArgs sig;
  CapArgs cap;
  int fuse_cap;  // single GPU: the warp completing the last signal applies the cap
};
#include "tail.cuh"  // k_tail: a2-a4 (+ a5-a7 in dsde_step)

template <typename KernelT>
static int resident_per_sm(KernelT k, int threads) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, 0);
  return std::max(1, per_sm);
}

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// Launch with programmatic dependent launch: the kernel may start while the
// previous kernel on the stream drains; it calls griddepcontrol.wait before
// touching that kernel's results.
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*kernel)(KArgs...), int grid, int block, cudaStream_t s, size_t dyn_smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = dyn_smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

// k_tail CTA shape: 32 warps while B <= SMs (one sequence per SM), 16 while
// B <= 2 SMs, else 8 (4 per SM, one wave up to B = 4 SMs).
template <typename T>
static void launch_tail(const TailArgs& p, int B, cudaStream_t s) {
  const int sms = sm_count();
  const size_t dyn = p.proposal ? sizeof(SpecRows) : 0;  // the D23 speculation records
  if (B <= sms) launch_pdl(k_tail<T, 32>, B, 1024, s, dyn, p);
  else if (B <= 2 * sms) launch_pdl(k_tail<T, 16>, B, 512, s, dyn, p);
  else launch_pdl(k_tail<T, 8>, std::min(B, 4 * sms), 256, s, dyn, p);
}

// step != nullptr: the whole-step launch (dsde_step) with the signal (and, if
// step->fuse_cap, the cap) in the tail kernel.
template <typename T>
cudaError_t launch_verify(int B, int V, int total, const int32_t* cu_sl, const int32_t* tokens,
                          const void* tl, int64_t ld_t, const void* dl, int64_t ld_d,
                          const uint64_t* seeds, int32_t* acc_len, int32_t* emitted, float* kld,
                          uint8_t* flags, const VerifyWs& ws, int32_t* err, Profiler* prof,
                          cudaStream_t s, const StepExtra* step = nullptr, int greedy = 0,
                          int dev_rows = 0, float* ent = nullptr, const float* temps = nullptr, int masked = 0,
                          int resample = DSDE_RESAMPLE_FULL) {
  const bool pr = prof != nullptr && prof->on;
  auto mark = [&]() {
    if (pr) cudaEventRecord(prof->next(), s);
  };
  const int ns = n_subs(V, sizeof(T) == 2 ? DSDE_BF16 : DSDE_F32);
  mark();
  // a1: the row stream (persistent warps; grid = resident CTAs)
  // D23 recovery draws (dsde_config.resample = DSDE_RESAMPLE_PROPOSAL, sampling modes)
  const bool proposal = resample == DSDE_RESAMPLE_PROPOSAL && !greedy;
  StreamArgs sa{tl, ld_t, dl, ld_d, cu_sl, B, V, ns, total, reinterpret_cast<SubPartial*>(ws.part), dev_rows,
                ws.counters, temps};
  const int sms = sm_count();
  auto go = [&](auto kern) {
    static int g = 0;  // one per instantiation
    if (!g) g = sms * resident_per_sm(kern, kLdgThreads);
    kern<<<g, kLdgThreads, 0, s>>>(sa);
  };
  if (masked) {
    if (dev_rows) go(k_stream_ldg<T, true, false, true>);
    else go(k_stream_ldg<T, false, false, true>);
  } else if (ent) {
    if (dev_rows) go(k_stream_ldg<T, true, true>);
    else go(k_stream_ldg<T, false, true>);
  } else {
    if (dev_rows) go(k_stream_ldg<T, true, false>);
    else go(k_stream_ldg<T, false, false>);
  }
  mark();
  // a2-a4 (+ a5-a7): the tail
  TailArgs p{};
  p.fa = FinArgs{B, V, total, ns, cu_sl, tokens, tl, ld_t, dl, ld_d, seeds,
                 reinterpret_cast<const SubPartial*>(ws.part), acc_len, emitted, kld, flags,
                 reinterpret_cast<SeqRec*>(ws.rec), err, greedy, dev_rows, ent, 0, temps, masked, ns, 0, nullptr};
  const int nd = n_draws(V, sizeof(T) == 2 ? DSDE_BF16 : DSDE_F32);
  p.sa = SelArgs{B, V, nd, tl, ld_t, dl, ld_d, emitted, flags, err, 0, 0, nd, V, nullptr};
  p.mass = ws.mass;
  p.mref = ws.mref;
  p.ctl = ws.counters;
  p.proposal = proposal;
  if (step) {
    p.step = 1;
    p.fuse_cap = step->fuse_cap;
    p.sig = step->sig;
    p.cap = step->cap;
  }
  launch_tail<T>(p, B, s);
  mark();
  mark();
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
  NvtxRange nv("dsde_verify");
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
  if ((long long)(total_draft_rows + B) * n_subs(V, dtype) > 0x3fffffffLL) return DSDE_ERR_ARG;
  if (st->cfg.masked && st->entropy_out) return DSDE_ERR_ARG;  // masks + draft entropy: not supported
  VerifyWs ws;
  ws_layout(B, total_draft_rows, V, dtype, &ws, reinterpret_cast<char*>(workspace));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (dtype == DSDE_BF16)
    e = launch_verify<uint16_t>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                                draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld,
                                flags, ws, st->err, st->prof, s, nullptr, st->cfg.greedy, st->cfg.device_rows,
                                st->entropy_out, st->temps, st->cfg.masked, st->cfg.resample);
  else
    e = launch_verify<float>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                             draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld, flags,
                             ws, st->err, st->prof, s, nullptr, st->cfg.greedy, st->cfg.device_rows,
                             st->entropy_out, st->temps, st->cfg.masked, st->cfg.resample);
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
  NvtxRange nv("dsde_step");
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
  if ((long long)(total_draft_rows + B) * n_subs(V, dtype) > 0x3fffffffLL) return DSDE_ERR_ARG;
  if (st->cfg.masked && st->entropy_out) return DSDE_ERR_ARG;        // masks + draft entropy: not supported
  if (st->cfg.entropy_mode && !st->entropy_out) return DSDE_ERR_ARG;  // D22 needs the draft entropy
  VerifyWs ws;
  ws_layout(B, total_draft_rows, V, dtype, &ws, reinterpret_cast<char*>(workspace));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  StepExtra x;
  x.sig = SignalArgs{st->cfg, B, st->max_seqs, slots, cu_sl, kld, accepted_len, sl_hat, diag,
                     st->seq, st->err, st->cfg.entropy_mode ? st->entropy_out : nullptr};
  x.cap = CapArgs{st->cfg, B, st->max_seqs, slots, sl_hat, budget, next_sl, cap, st->seq, st->scratch};
  x.fuse_cap = comm == nullptr;
  cudaError_t e;
  if (dtype == DSDE_BF16)
    e = launch_verify<uint16_t>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                                draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld,
                                flags, ws, st->err, st->prof, s, &x, st->cfg.greedy, st->cfg.device_rows,
                                st->entropy_out, st->temps, st->cfg.masked, st->cfg.resample);
  else
    e = launch_verify<float>(B, V, total_draft_rows, cu_sl, draft_tokens, target_logits, ld_t,
                             draft_logits, ld_d, seeds, accepted_len, emitted_tokens, kld, flags,
                             ws, st->err, st->prof, s, &x, st->cfg.greedy, st->cfg.device_rows,
                             st->entropy_out, st->temps, st->cfg.masked, st->cfg.resample);
  if (e != cudaSuccess) return DSDE_ERR_CUDA;
  if (!comm) return DSDE_OK;
  dsde_status rs = DSDE_OK;
  e = launch_cap_multi(x.cap, comm, s, &rs);
  if (rs != DSDE_OK) return rs;
  return e == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}


#include "vocab.cuh"  // vocab-parallel verification stages

#if DSDE_TAIL_TRACE
// measurement build only: copy the k_tail trace (8 u64 per CTA)
extern "C" int dsde_debug_tail_trace(unsigned long long* out, int n) {
  n = n < dsde::kTraceMax ? n : dsde::kTraceMax;
  return cudaMemcpyFromSymbol(out, dsde::g_tail_trace, sizeof(unsigned long long) * 8 * n) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" dsde_status dsde_set_draft_entropy(dsde_state st, float* entropy) {
  if (!st) return DSDE_ERR_ARG;
  st->entropy_out = entropy;
  return DSDE_OK;
}

extern "C" dsde_status dsde_set_temperature(dsde_state st, const float* temperature) {
  if (!st) return DSDE_ERR_ARG;
  st->temps = temperature;
  return DSDE_OK;
}

