// verify_draw.cuh — a2-a4 of dsde_verify after the stream pass (included by
// verify.cu inside namespace dsde; uses its helpers).
//
//   k_finalize  one CTA per sequence, one warp per draft position: fp64 merge of
//               the row's slice partials (lanes over slices), KL, log p/q; then
//               warp 0 runs the Philox accept test of every position, finds the
//               first rejection a_i, lays out the emitted tokens and publishes
//               the draw record (residual row a_i, or the bonus row k_i) (a2-a3).
//   k_draw_*    every warp forms the draw weights of one 1024-token (bf16) /
//               512-token (fp32) slice of the drawn row and writes their mass
//               (a4, first pass); persistent warps as k_stream_ldg.
//   k_select    one warp per sequence: the inverse CDF over the slice masses,
//               then inside the crossing slice (re-read from L2)
//               in ascending token order (a4, D7).

enum { IT_RESID = 1, IT_BONUS = 2, IT_NONE = 3, IT_ARGMAX = 4 };

struct FinArgs {
  int B, V, total, nsub;
  const int32_t* cu_sl;
  const int32_t* tokens;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const uint64_t* seeds;
  const SubPartial* part;
  int32_t* acc_len;
  int32_t* emitted;
  float* kld;
  uint8_t* flags;
  SeqRec* rec;
  int32_t* err;
  int greedy;  // T = 0: accept iff x = argmax t, emit the argmax
  int dev_rows;  // dsde_config.device_rows: total is a capacity, Σk_i = cu_sl[B]
  float* ent;    // [Σk_i] optional out: draft entropy H(q) per row; partials carry Sd, E
};

constexpr int kFinThreads = 32 * DSDE_MAX_SL;

// One CTA (kFinThreads) per sequence i; the draw record goes to *out (global
// or shared; written by one lane of warp 0, visible to the CTA after a barrier).
// Warp 0's per-position inputs of the accept test (lane j = position j): the
// Philox uniforms and the gathered t_x, d_x. They depend only on the step's
// inputs, so k_tail gathers them before griddepcontrol.wait, while the stream
// kernel still runs (the inputs were complete before the stream kernel began).
struct FinPre {
  Uniforms u;
  float tx, dx;
  int x;
};

template <typename T>
__device__ __forceinline__ FinPre fin_prefetch(const FinArgs& a, int i) {
  const int lane = threadIdx.x & 31;
  FinPre p;
  p.u = Uniforms{0.0, 0.0};
  p.tx = p.dx = 0.f;
  p.x = -1;
  const int c0 = __ldg(a.cu_sl + i), c1 = __ldg(a.cu_sl + i + 1);
  const int k = c1 - c0;
  if (!(c0 >= 0 && k >= 1 && k <= DSDE_MAX_SL && c1 <= a.total)) return p;  // finalize_seq reports it
  const long long slot0 = (long long)c0 + i;
  if (lane <= k) p.u = philox_uniforms(__ldg(a.seeds + slot0 + lane));
  if (lane < k) {
    const long long drow = (long long)c0 + lane;
    p.x = __ldg(a.tokens + drow);
    if (p.x >= 0 && p.x < a.V) {
      p.tx = load_logit<T>(reinterpret_cast<const T*>(a.tl) + (drow + i) * a.ld_t + p.x);
      p.dx = load_logit<T>(reinterpret_cast<const T*>(a.dl) + drow * a.ld_d + p.x);
    }
  }
  return p;
}

// pre: warp 0's fin_prefetch results (k_tail), or nullptr to load them here.
template <typename T>
__device__ __forceinline__ void finalize_seq(const FinArgs& a, int i, SeqRec* out, const FinPre* pre = nullptr) {
  __shared__ double s_kl[DSDE_MAX_SL], s_lam[DSDE_MAX_SL], s_C[DSDE_MAX_SL], s_S[DSDE_MAX_SL];
  __shared__ int s_amax[DSDE_MAX_SL];
  __shared__ float s_M[DSDE_MAX_SL];
  __shared__ int s_fin[DSDE_MAX_SL];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = __ldg(a.cu_sl + i), c1 = __ldg(a.cu_sl + i + 1);
  const int k = c1 - c0;
  const bool range_ok = c0 >= 0 && k >= 1 && k <= DSDE_MAX_SL && c1 <= a.total;
  const bool rows_ok = a.dev_rows || (i != a.B - 1) || (c1 == a.total);
  if (!range_ok || !rows_ok) {
    if (threadIdx.x == 0) {
      a.acc_len[i] = -1;
      out->mode = MODE_ERROR;
      raise_device_error(a.err, range_ok ? DSDE_DERR_ROWS : DSDE_DERR_BAD_SL, i);
    }
    return;
  }
  const int nc = a.nsub;
  const int nwarps = blockDim.x >> 5;
  for (int j = warp; j < k; j += nwarps) {
    // ---- row j: fp64 merge of the slice partials (lanes over slices c)
    // about M = max_c M_c, C = fp32(M - max d). Slice c's w is shifted by
    // Delta = C_c - C; with s = e^(M_c - M), E1 = s e^-Delta:
    //   S += s S_c,  A += s (A_c + S_c Delta),
    //   D += E1 D_c - A_c s expm1(-Delta) + S_c s g(Delta),  g(x) = expm1(-x) + x.
    const SubPartial* P = a.part + ((long long)c0 + j) * nc;
    float Ml = -INFINITY, Dl = -INFINITY;
    for (int c = lane; c < nc; c += 32) {
      Ml = max_nan(Ml, P[c].M);
      Dl = fmaxf(Dl, P[c].maxd);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Ml = max_nan(Ml, __shfl_xor_sync(kFull, Ml, o));
      Dl = fmaxf(Dl, __shfl_xor_sync(kFull, Dl, o));
    }
    const double M = (double)Ml, C = (double)(Ml - Dl);  // C is an fp32 value
    double S = 0.0, A = 0.0, D = 0.0, Sd = 0.0, E = 0.0;
    for (int c = lane; c < nc; c += 32) {
      const float4 q0 = __ldg(reinterpret_cast<const float4*>(P + c));
      const float4 q1 = __ldg(reinterpret_cast<const float4*>(P + c) + 1);
      const double qS = q0.x, qA = q0.y, qD = q0.z, qM = q0.w, qC = q1.x;
      if (a.ent && q1.z > 0.f) {
        // draft sums about the row max of d: Sd += s Sd_c, E += s (E_c + (maxd_c - maxd) Sd_c)
        const double dd = (double)q1.y - (double)Dl, sd = exp(dd);
        Sd += sd * (double)q1.z;
        E += sd * ((double)q1.w + dd * (double)q1.z);
      }
      const double ls = qM - M;
      const double s = exp(ls);
      const double dl = qC - C;
      double sem, sg, E1;
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
      S += s * qS;
      A += s * qA + s * qS * dl;
      D += E1 * qD - qA * sem + qS * sg;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      S += __shfl_xor_sync(kFull, S, o);
      A += __shfl_xor_sync(kFull, A, o);
      D += __shfl_xor_sync(kFull, D, o);
    }
    if (a.ent) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        Sd += __shfl_xor_sync(kFull, Sd, o);
        E += __shfl_xor_sync(kFull, E, o);
      }
      // H(q) = log Sd - E / Sd (E <= 0: both terms non-negative, no cancellation)
      if (lane == 0) a.ent[c0 + j] = (float)(log(Sd) - E / Sd);
    }
    if (a.greedy) {
      // row argmax of t: the first slice holding the row max (slices are in
      // token order), re-read from memory vector by vector (token order is
      // vector-major) until a lane holds the max; its first such element
      constexpr int VEC = Traits<T>::VEC, SUB = sub_elems<T>();
      unsigned cs = 0x7fffffffu;
      for (int c = lane; c < nc; c += 32)
        if (P[c].M == Ml) cs = min(cs, (unsigned)c);
      cs = __reduce_min_sync(kFull, cs);
      int amax = 0x7fffffff;
      if (cs < (unsigned)nc) {
        const T* trow = reinterpret_cast<const T*>(a.tl) + ((long long)c0 + i + j) * a.ld_t + cs * SUB;
        const int left = a.V - (int)cs * SUB;
        for (int v = 0; v * 32 * VEC < min(SUB, left); ++v) {
          const int e0 = (v * 32 + lane) * VEC;
          int first = 0x7fffffff;
#pragma unroll
          for (int e = VEC - 1; e >= 0; --e)
            if (e0 + e < left && load_logit<T>(trow + e0 + e) == Ml) first = e0 + e;
          const unsigned hit = __ballot_sync(kFull, first != 0x7fffffff);
          if (hit) {
            amax = (int)cs * SUB + __shfl_sync(kFull, first, __ffs(hit) - 1);
            break;
          }
        }
      }
      if (lane == 0) s_amax[j] = amax;
    }
    if (lane == 0) {
      // y = E_p[exp(-w)] - 1. KL = D/S + (log1p(y) - y) has no cancellation for
      // small KL; when y > 1 (the draft puts far more mass away from the
      // reference, e.g. disjoint supports) the equal form A/S + log1p(y) is used.
      const double y = (D - A) / S;
      const double lam = log1p(y);
      const double kl = fmax(0.0, y <= 1.0 ? D / S + (lam - y) : A / S + lam);
      s_kl[j] = kl;
      s_lam[j] = lam;
      s_C[j] = C;
      s_M[j] = Ml;
      s_S[j] = S;
      s_fin[j] = isfinite(S) && isfinite(A) && isfinite(D) && S > 0.0 && isfinite(M) &&
                    isfinite(C) && isfinite(kl);
    }
  }
  __syncthreads();
  if (warp != 0) return;
  // ---- warp 0, lane j = position j: accept test, first rejection, layout ----
  const long long slot0 = (long long)c0 + i;
  double lr = 0.0;
  bool acc = false, near = false, bad_tok = false, nonfin = false;
  Uniforms u = {0.0, 0.0};
  if (pre) u = pre->u;
  else if (lane <= k) u = philox_uniforms(__ldg(a.seeds + slot0 + lane));
  if (lane < k) {
    const long long drow = (long long)c0 + lane;
    const int x = pre ? pre->x : __ldg(a.tokens + drow);
    bad_tok = x < 0 || x >= a.V;
    nonfin = !s_fin[lane];
    if (!bad_tok) {
      const T* tp = reinterpret_cast<const T*>(a.tl) + (drow + i) * a.ld_t;
      const T* dp = reinterpret_cast<const T*>(a.dl) + drow * a.ld_d;
      const double tx = (double)(pre ? pre->tx : load_logit<T>(tp + x));
      const double dx = (double)(pre ? pre->dx : load_logit<T>(dp + x));
      lr = (tx - dx) - s_C[lane] + s_lam[lane];
      nonfin |= !isfinite(lr);
    }
    if (a.greedy) {
      acc = x == s_amax[lane];  // T = 0: the draft token must be the target argmax
    } else {
      const double pacc = lr >= 0.0 ? 1.0 : exp(lr);
      acc = u.acc < pacc;
      near = fabs(u.acc - pacc) < 1e-6;
    }
  }
  const unsigned bt = __ballot_sync(kFull, bad_tok);
  const unsigned nf = __ballot_sync(kFull, nonfin);
  const unsigned am = __ballot_sync(kFull, acc);
  SeqRec r;
  r.pad0 = 0;
  r.S = 0.0;
  if (bt | nf) {
    if (lane < k) a.kld[c0 + lane] = NAN;
    if (lane <= k) {
      a.emitted[slot0 + lane] = DSDE_PAD;
      if (a.flags) a.flags[slot0 + lane] = 0;
    }
    if (lane == 0) {
      a.acc_len[i] = -1;
      raise_device_error(a.err, bt ? DSDE_DERR_BAD_TOKEN : DSDE_DERR_NONFINITE, i);
      r.mode = MODE_ERROR;
      r.slot = (int)slot0;
      r.trow = slot0;
      r.drow = -1;
      r.M = 0.f;
      r.C = r.lam = r.u = 0.0;
      *out = r;
    }
    return;
  }
  const int acc_run = __ffs(~am) - 1;  // first rejected lane (lanes >= k never accept)
  const int aa = acc_run < k ? acc_run : k;
  if (lane < k) a.kld[c0 + lane] = (float)s_kl[lane];
  if (lane <= k) {
    a.emitted[slot0 + lane] = lane < aa ? __ldg(a.tokens + c0 + lane) : DSDE_PAD;
    if (a.flags) a.flags[slot0 + lane] = (near && lane <= aa && lane < k) ? DSDE_FLAG_ACCEPT_NEAR_TIE : 0;
  }
  if (lane == 0) a.acc_len[i] = aa;
  if (lane == aa && a.greedy) {
    // T = 0: the recovery token is the argmax of row aa (known from the stream);
    // the bonus row's argmax is found by the draw pass
    r.slot = (int)(slot0 + aa);
    r.trow = slot0 + aa;
    r.drow = -1;
    r.u = 0.0;
    r.M = 0.f;
    r.C = r.lam = 0.0;
    if (aa < k) {
      a.emitted[slot0 + aa] = s_amax[aa];
      r.mode = MODE_NONE;
    } else {
      r.mode = MODE_ARGMAX;
    }
    *out = r;
  } else if (lane == aa) {
    r.slot = (int)(slot0 + aa);
    r.trow = slot0 + aa;
    r.u = u.smp;
    if (aa < k) {
      r.mode = MODE_RESIDUAL;
      r.drow = (long long)c0 + aa;
      r.M = s_M[aa];
      r.C = s_C[aa];
      r.lam = s_lam[aa];
      r.S = s_S[aa];
    } else {
      r.mode = MODE_BONUS;
      r.drow = -1;
      r.M = 0.f;
      r.C = 0.0;
      r.lam = 0.0;
    }
    *out = r;
  }
}

template <typename T>
__global__ void __launch_bounds__(kFinThreads) k_finalize(FinArgs a) {
  finalize_seq<T>(a, blockIdx.x, a.rec + blockIdx.x);
}

// ---------------------------------------------------------------------------
// draw weights of one lane over a 1024-token (bf16) / 512-token (fp32)
// sub-chunk u, token u*SUB + (v*32 + lane)*VEC + e, from raw words; returns the
// reference (residual: M of the row; bonus: warp max of t).
//   residual: rho_v = e_v (1 - exp(-z_v)) for z_v > 0, else 0, with
//             e_v = exp(t_v - M), z_v = w_v + lam, w_v = (t_v - d_v) - C exact,
//             lam added as hi + lo floats; 1 - exp(-z) = z (1 - z h(-z)) for
//             z < 1 (no cancellation), 1 - 2^(-z log2 e) otherwise;
//   bonus:    p_v up to a scale: exp(t_v - m_u) about the warp max m_u,
//             rescaled by exp(m_u - max_u m_u) in fp64 by k_select.
// The select recomputes every weight bit-identically from the same words.
// ---------------------------------------------------------------------------
// degree of the h(-z) fit on |z| < 1 in the residual weights
#ifndef DSDE_RESID_DEG
#define DSDE_RESID_DEG 6
#endif
// residual weights of one element pair (see above)
template <typename T>
__device__ __forceinline__ float2 resid_pair_exact(float2 tt, float2 dd, float2 nML2, float khi, float klo) {
  const float2 L2 = make_float2(kLog2e, kLog2e), nL2 = make_float2(-kLog2e, -kLog2e);
  const float2 ONE = make_float2(1.f, 1.f);
#if DSDE_RESID_DEG == 7  // degree 7 on |z| <= 1 (1.1e-7 relative)
  const float2 K7 = make_float2(-2.812654656736413e-06f, -2.812654656736413e-06f);
  const float2 K6 = make_float2(2.5358644052175805e-05f, 2.5358644052175805e-05f);
  const float2 K5 = make_float2(-1.9836986029986292e-04f, -1.9836986029986292e-04f);
  const float2 K4 = make_float2(1.3885394437238574e-03f, 1.3885394437238574e-03f);
  const float2 K3 = make_float2(-8.33334494382143e-03f, -8.33334494382143e-03f);
  const float2 K2 = make_float2(4.166673496365547e-02f, 4.166673496365547e-02f);
  const float2 K1 = make_float2(-1.666666716337204e-01f, -1.666666716337204e-01f);
#else  // degree 6 on |z| <= 1 (2.0e-7 relative; the stream's exact-path fit)
  const float2 K6 = make_float2(2.5358644052175805e-05f, 2.5358644052175805e-05f);
  const float2 K5 = make_float2(-2.0329201652202755e-04f, -2.0329201652202755e-04f);
  const float2 K4 = make_float2(1.3885394437238574e-03f, 1.3885394437238574e-03f);
  const float2 K3 = make_float2(-8.330884389579296e-03f, -8.330884389579296e-03f);
  const float2 K2 = make_float2(4.166673496365547e-02f, 4.166673496365547e-02f);
  const float2 K1 = make_float2(-1.6666696965694427e-01f, -1.6666696965694427e-01f);
#endif
  const float2 K0 = make_float2(0.5f, 0.5f);
  const float2 xt = __ffma2_rn(tt, L2, nML2);
  const float2 ev = make_float2(fast_exp2(xt.x), fast_exp2(xt.y));  // 0 for padding
  // z = (t - d) - (C - lam), the constant carried as khi + klo
  float2 z;
  if constexpr (sizeof(T) == 2) {
    z = __fadd2_rn(__fadd2_rn(tt, make_float2(-dd.x, -dd.y)), make_float2(-khi, -khi));  // t - d exact
  } else {
    z = make_float2(diff_ref<T>(tt.x, dd.x, khi), diff_ref<T>(tt.y, dd.y, khi));
  }
  z = __fadd2_rn(z, make_float2(-klo, -klo));
#if DSDE_RESID_DEG == 7
  float2 pz = __ffma2_rn(K7, z, K6);
  pz = __ffma2_rn(pz, z, K5);
#else
  float2 pz = __ffma2_rn(K6, z, K5);
#endif
  pz = __ffma2_rn(pz, z, K4);
  pz = __ffma2_rn(pz, z, K3);
  pz = __ffma2_rn(pz, z, K2);
  pz = __ffma2_rn(pz, z, K1);
  pz = __ffma2_rn(pz, z, K0);
  const float2 sm = __fmul2_rn(z, __ffma2_rn(make_float2(-z.x, -z.y), pz, ONE));  // z (1 - z h(-z))
  const float2 xz = __fmul2_rn(z, nL2);
  const float2 bg = __fadd2_rn(ONE, make_float2(-fast_exp2(xz.x), -fast_exp2(xz.y)));  // 1 - e^-z
  // 1 - e^-z <= 0 for z <= 0 in both forms (the polynomial only on |z| < 1),
  // so max(0, .) zeroes exactly the tokens with p_v <= q_v (fmaxf drops the NaN
  // of padding, 0 * -inf)
  const float2 om = make_float2(fabsf(z.x) < 1.f ? sm.x : bg.x, fabsf(z.y) < 1.f ? sm.y : bg.y);
  const float2 r = __fmul2_rn(ev, om);
  return make_float2(fmaxf(r.x, 0.f), fmaxf(r.y, 0.f));
}

// lane max of t over one vector (NaN-propagating)
template <typename T>
__device__ __forceinline__ float vec_tmax(const uint4& t, float m) {
  const uint4 x[1] = {t};
#pragma unroll
  for (int h = 0; h < Traits<T>::VEC; h += 2) {
    const float2 tt = pair_of<T>(x, h);
    m = max_nan(m, max_nan(tt.x, tt.y));
  }
  return m;
}

// Per-slice constants of the draw weights.
struct DrawRef {
  bool resid;
  float M, khi, klo;  // residual: row reference M, C - lam = khi + klo
  float m;            // bonus: the slice's warp max of t (reference)
};

// Warp-wide max of t over a lane's NV vectors (NaN-propagating; packed
// max.NaN.bf16x2 for bf16: max is exact, so any grouping gives the same value).
template <typename T, int NV>
__device__ __forceinline__ float slice_tmax(const uint4 (&rt)[NV]) {
  float m;
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162 b0 = __floats2bfloat162_rn(-INFINITY, -INFINITY), b1 = b0;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const uint32_t w4[4] = {rt[v].x, rt[v].y, rt[v].z, rt[v].w};
      b0 = __hmax2_nan(b0, *reinterpret_cast<const __nv_bfloat162*>(&w4[0]));
      b1 = __hmax2_nan(b1, *reinterpret_cast<const __nv_bfloat162*>(&w4[1]));
      b0 = __hmax2_nan(b0, *reinterpret_cast<const __nv_bfloat162*>(&w4[2]));
      b1 = __hmax2_nan(b1, *reinterpret_cast<const __nv_bfloat162*>(&w4[3]));
    }
    const __nv_bfloat162 b = __hmax2_nan(b0, b1);
    m = max_nan(__low2float(b), __high2float(b));
  } else {
    m = -INFINITY;
#pragma unroll
    for (int v = 0; v < NV; ++v) m = vec_tmax<T>(rt[v], m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max_nan(m, __shfl_xor_sync(kFull, m, o));
  return m;
}

// Slice constants; for the bonus row the warp-wide max of t over the slice.
template <typename T, int NV>
__device__ __forceinline__ DrawRef draw_ref(const uint4 (&rt)[NV], bool resid, float M, float Cf, double lam) {
  DrawRef R;
  R.resid = resid;
  R.M = M;
  const double K = (double)Cf - lam;
  R.khi = (float)K;
  R.klo = (float)(K - (double)R.khi);
  R.m = resid ? 0.f : slice_tmax<T, NV>(rt);
  return R;
}

// Draw weights of the VEC tokens of one lane vector.
template <typename T>
__device__ __forceinline__ void vec_weights(const uint4& t4, const uint4& d4, const DrawRef& R,
                                            float (&w)[Traits<T>::VEC]) {
  constexpr int VEC = Traits<T>::VEC;
  const uint4 rt[1] = {t4}, rd[1] = {d4};
  const float2 L2 = make_float2(kLog2e, kLog2e);
  if (R.resid) {
    const float ML2 = R.M * kLog2e;
    const float2 nML2 = make_float2(-ML2, -ML2);
#pragma unroll
    for (int h = 0; h < VEC; h += 2) {
      const float2 r = resid_pair_exact<T>(pair_of<T>(rt, h), pair_of<T>(rd, h), nML2, R.khi, R.klo);
      w[h] = r.x;
      w[h + 1] = r.y;
    }
    return;
  }
  if (R.m <= -1e30f) {  // an all-padding slice (warp-uniform)
#pragma unroll
    for (int e = 0; e < VEC; ++e) w[e] = 0.f;
    return;
  }
  const float mL2 = R.m * kLog2e;
  const float2 nmL2 = make_float2(-mL2, -mL2);
#pragma unroll
  for (int h = 0; h < VEC; h += 2) {
    const float2 x = __ffma2_rn(pair_of<T>(rt, h), L2, nmL2);
    w[h] = fast_exp2(x.x);
    w[h + 1] = fast_exp2(x.y);
  }
}

// raw words of sub-chunk u of a row, from global memory (select pass)
template <typename T, int NV>
__device__ __forceinline__ void load_sub_raw(const T* row, int V, int u, uint4 (&r)[NV]) {
  constexpr int VEC = Traits<T>::VEC, SUB = 32 * VEC * NV;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int e0 = u * SUB + (v * 32 + lane) * VEC;
    if (e0 + VEC <= V) {
      r[v] = __ldcg(reinterpret_cast<const uint4*>(row + e0));
    } else {
      T b[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) b[e] = (e0 + e < V) ? row[e0 + e] : pad_bits<T>();
      r[v] = *reinterpret_cast<const uint4*>(b);
    }
  }
}

__device__ __forceinline__ double wsum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__device__ __forceinline__ double wscan_d(double x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// sum_v (sum over the 32 lanes of x[v]) in vector order, valid in lane 0: the
// NV per-vector warp sums by recursive halving (the first log2(NV) butterfly
// rounds exchange half of the remaining vectors, so each round moves one
// double per kept vector instead of one per vector), lanes 8 j .. hold vector
// j's total (NV = 4), then lane 0 gathers them.
template <int NV>
__device__ __forceinline__ double warp_sum_vectors(double (&x)[NV]) {
  static_assert(NV == 1 || NV == 2 || NV == 4 || NV == 8, "NV");
  const int lane = threadIdx.x & 31;
  int o = 16;
#pragma unroll
  for (int cnt = NV; cnt > 1; cnt >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < cnt / 2; ++j) {
      const double send = up ? x[j] : x[j + cnt / 2];
      const double keep = up ? x[j + cnt / 2] : x[j];
      x[j] = keep + __shfl_xor_sync(kFull, send, o);
    }
  }
#pragma unroll
  for (; o > 0; o >>= 1) x[0] += __shfl_xor_sync(kFull, x[0], o);
  // vector index of lane l's total: bit (log2 NV - 1 - b) of it is bit (4 - b) of l
  double m = 0.0;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    int src = 0;
#pragma unroll
    for (int b = 0, n = NV; n > 1; ++b, n >>= 1)
      if (v & (n >> 1)) src |= 16 >> b;
    m += __shfl_sync(kFull, x[0], src);
  }
  return m;
}

// ---------------------------------------------------------------------------
// a4 first pass: units q = (sequence i, slice u), q = i * nsub + u. Each warp
// writes the mass of its slice's draw weights and the slice reference.
// ---------------------------------------------------------------------------
struct DrawArgs {
  int B, V, nsub;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const SeqRec* rec;
  double* smass;  // [B * nsub]
  float* sref;    // [B * nsub]
};

struct DrawUnit {
  int type;  // IT_RESID / IT_BONUS / IT_NONE
  float M, Cf;
  double lam;
};

template <typename T>
__device__ __forceinline__ DrawUnit draw_unit_load(const DrawArgs& a, int u, const SeqRec& r,
                                                   uint4 (&rt)[Traits<T>::NVD], uint4 (&rd)[Traits<T>::NVD]) {
  const int mode = r.mode;
  DrawUnit d;
  d.type = mode == MODE_RESIDUAL ? IT_RESID : mode == MODE_BONUS ? IT_BONUS : mode == MODE_ARGMAX ? IT_ARGMAX : IT_NONE;
  d.M = 0.f;
  d.Cf = 0.f;
  d.lam = 0.0;
  if (d.type == IT_NONE) return d;
  load_slice<T>(reinterpret_cast<const T*>(a.tl) + r.trow * a.ld_t, a.V, u, rt);
  if (d.type == IT_RESID) {
    load_slice<T>(reinterpret_cast<const T*>(a.dl) + r.drow * a.ld_d, a.V, u, rd);
    d.M = r.M;
    d.Cf = (float)r.C;
    d.lam = r.lam;
  }
  return d;
}

template <typename T>
__device__ __forceinline__ DrawUnit draw_unit_load(const DrawArgs& a, long long q, uint4 (&rt)[Traits<T>::NVD],
                                                   uint4 (&rd)[Traits<T>::NVD]) {
  const SeqRec* rp = a.rec + (int)(q / a.nsub);
  SeqRec r;
  r.mode = __ldg(&rp->mode);
  if (r.mode == MODE_RESIDUAL || r.mode == MODE_BONUS || r.mode == MODE_ARGMAX) {
    r.trow = __ldg(&rp->trow);
    r.drow = __ldg(&rp->drow);
    r.M = __ldg(&rp->M);
    r.C = __ldg(&rp->C);
    r.lam = __ldg(&rp->lam);
  }
  return draw_unit_load<T>(a, (int)(q - (q / a.nsub) * a.nsub), r, rt, rd);
}

// mass_out / ref_out: this unit's record (global a.smass + q, or the k_tail
// CTA's shared arrays)
template <typename T>
__device__ __forceinline__ void draw_unit_finish(double* mass_out, float* ref_out, const DrawUnit& d,
                                                 const uint4 (&rt)[Traits<T>::NVD],
                                                 const uint4 (&rd)[Traits<T>::NVD]) {
  constexpr int VEC = Traits<T>::VEC, NVD = Traits<T>::NVD;
  if (d.type == IT_NONE) return;
  if (d.type == IT_ARGMAX) {
    // greedy bonus row: the slice max of t and its first (slice-local) index
    const int lane = threadIdx.x & 31;
    const float m = slice_tmax<T, NVD>(rt);
    int best = 0x7fffffff;
#pragma unroll
    for (int v = NVD - 1; v >= 0; --v) {
      const uint4 x[1] = {rt[v]};
#pragma unroll
      for (int h = VEC - 2; h >= 0; h -= 2) {
        const float2 tt = pair_of<T>(x, h);
        const int e0 = (v * 32 + lane) * VEC + h;
        if (tt.y == m) best = e0 + 1;
        if (tt.x == m) best = e0;
      }
    }
    best = (int)__reduce_min_sync(kFull, (unsigned)best);
    if (lane == 0) {
      *mass_out = (double)best;
      *ref_out = m;
    }
    return;
  }
  const DrawRef R = draw_ref<T>(rt, d.type == IT_RESID, d.M, d.Cf, d.lam);
  // mass in the select pass's grouping: per vector an fp32 lane sum, an fp64
  // sum over the 32 lanes, the vectors added in order
  double x[NVD];
#pragma unroll
  for (int v = 0; v < NVD; ++v) {
    float w[VEC];
    vec_weights<T>(rt[v], rd[v], R, w);
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += w[e];
    x[v] = (double)ls;
  }
  const double m = warp_sum_vectors<NVD>(x);
  if ((threadIdx.x & 31) == 0) {
    *mass_out = m;
    *ref_out = R.resid ? R.M : (R.m <= -1e30f ? -INFINITY : R.m);
  }
}

// "ldg" variant: persistent warps, the next unit's vectors in flight while the
// current one is computed (as k_stream_ldg).
#ifndef DSDE_DRAW_MINB
#define DSDE_DRAW_MINB 3
#endif
template <typename T>
__global__ void __launch_bounds__(kLdgThreads, DSDE_DRAW_MINB) k_draw_ldg(DrawArgs a) {
  constexpr int NV = Traits<T>::NVD;
  const long long n_units = (long long)a.B * a.nsub;
  const long long W = (long long)gridDim.x * (kLdgThreads / 32);
  long long q = (long long)blockIdx.x * (kLdgThreads / 32) + (threadIdx.x >> 5);
  if (q >= n_units) return;
  for (; q < n_units; q += W) {
    uint4 rt[NV], rd[NV];
    const DrawUnit d = draw_unit_load<T>(a, q, rt, rd);
    draw_unit_finish<T>(a.smass + q, a.sref + q, d, rt, rd);
  }
}

// ---------------------------------------------------------------------------
// k_select: one warp per sequence (4 per CTA).
// ---------------------------------------------------------------------------
struct SelArgs {
  int B, V, nsub;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const SeqRec* rec;
  const double* smass;
  const float* sref;
  int32_t* emitted;
  uint8_t* flags;
  int32_t* err;
};

#ifndef DSDE_TAIL_TRACE
#define DSDE_TAIL_TRACE 0
#endif
#if DSDE_TAIL_TRACE
// measurement build only (-DDSDE_TAIL_TRACE=1): per-CTA globaltimer stamps at
// the phase boundaries of k_tail, read back by dsde_debug_tail_trace
constexpr int kTraceMax = 4096;
__device__ unsigned long long g_tail_trace[kTraceMax * 6];
__device__ __forceinline__ void tail_stamp(int slot, unsigned long long v) {
  if (threadIdx.x == 0 && blockIdx.x < kTraceMax) g_tail_trace[blockIdx.x * 6 + slot] = v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define TAIL_STAMP(slot) tail_stamp(slot, gtimer())
#else
#define TAIL_STAMP(slot)
#endif

// Where select_seq reads the slice records from: global memory written by
// another kernel / CTA (masses about each slice's own reference, rescaled
// here), or the k_tail CTA's shared arrays with the bonus masses already
// rescaled to the row reference by the whole CTA (scale[] = the factors).
struct SelSrcGlobal {
  static constexpr bool kPrescaled = false;
  const double* m;
  const float* r;
  __device__ __forceinline__ double mass(int s) const { return __ldcg(m + s); }
  __device__ __forceinline__ float ref(int s) const { return __ldcg(r + s); }
  __device__ __forceinline__ double scale(int) const { return 1.0; }
};
struct SelSrcSmem {
  static constexpr bool kPrescaled = true;
  const double* m;
  const float* r;
  const double* sc;
  __device__ __forceinline__ double mass(int s) const { return m[s]; }
  __device__ __forceinline__ float ref(int s) const { return r[s]; }
  __device__ __forceinline__ double scale(int s) const { return sc[s]; }
};

// One warp: the inverse-CDF select of sequence i from its slice masses.
template <typename T, typename Src>
__device__ __forceinline__ void select_seq(const SelArgs& a, int i, const SeqRec& r, const Src& src) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NVD, SUB = 32 * VEC * NV;
  const int lane = threadIdx.x & 31;
  if (r.mode == MODE_ARGMAX) {
    // greedy bonus token: the smallest index among the slices holding the row max
    float Mg = -INFINITY;
    for (int s0 = lane; s0 < a.nsub; s0 += 32) Mg = max_nan(Mg, src.ref(s0));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mg = max_nan(Mg, __shfl_xor_sync(kFull, Mg, o));
    unsigned cand = 0x7fffffffu;
    for (int s0 = lane; s0 < a.nsub; s0 += 32)
      if (src.ref(s0) == Mg) cand = min(cand, (unsigned)(s0 * SUB + (int)src.mass(s0)));
    cand = __reduce_min_sync(kFull, cand);
    if (lane == 0) {
      if (Mg != Mg || cand >= (unsigned)a.V) {
        a.emitted[r.slot] = DSDE_PAD;
        raise_device_error(a.err, DSDE_DERR_NONFINITE, i);
      } else {
        a.emitted[r.slot] = (int)cand;
      }
    }
    return;
  }
  if (r.mode != MODE_RESIDUAL && r.mode != MODE_BONUS) return;
  const bool resid = r.mode == MODE_RESIDUAL;
  const int nsub = a.nsub;
  float Mg = -INFINITY;
  if (!resid && !Src::kPrescaled) {
    for (int s0 = lane; s0 < nsub; s0 += 32) Mg = max_nan(Mg, src.ref(s0));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mg = max_nan(Mg, __shfl_xor_sync(kFull, Mg, o));
  }
  auto scale_of = [&](int s0) -> double {  // sub-chunk mass scale to the common reference
    if (resid) return 1.0;
    if constexpr (Src::kPrescaled) {
      return src.scale(s0);
    } else {
      const float ms = src.ref(s0);
      return ms == -INFINITY ? 0.0 : exp((double)ms - (double)Mg);
    }
  };
  auto mass_of = [&](int s0) -> double {  // scale_of(s0) * the slice's own mass
    if constexpr (Src::kPrescaled) return src.mass(s0);
    else return scale_of(s0) * src.mass(s0);
  };
  // lane l owns the contiguous slices [l c, (l + 1) c): its sum in slice order,
  // one warp scan gives every lane's prefix and R (the scan's total)
  const int cw = (nsub + 31) >> 5;
  const int s_lo = min(lane * cw, nsub), s_hi = min(s_lo + cw, nsub);
  double lsum = 0.0;
  for (int s0 = s_lo; s0 < s_hi; ++s0) lsum += mass_of(s0);
  const double lincl = wscan_d(lsum, lane);
  const double R = __shfl_sync(kFull, lincl, 31);
  uint8_t fl = 0;
  const T* tp = reinterpret_cast<const T*>(a.tl) + r.trow * a.ld_t;
  if (!(R > 0.0) || !isfinite(R)) {
    if (lane == 0) {
      // residual mass 0 (p <= q everywhere in fp32; D7 fallback: draw from p
      // of the same target row, one lane) or a non-finite bonus row
      if (resid && isfinite(R)) {
        double tot = 0.0;
        for (int v = 0; v < a.V; ++v) tot += exp((double)load_logit<T>(tp + v) - (double)r.M);
        const double target = r.u * tot;
        double cum = 0.0;
        int tok = 0;
        for (int v = 0; v < a.V; ++v) {
          const double wv = exp((double)load_logit<T>(tp + v) - (double)r.M);
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
  // crossing sub-chunk: first u with prefix(u) > target (fallback: last with
  // mass): the first lane whose span crosses, then that lane's slices in order
  int us = -1;
  double base = 0.0;
  {
    double lexcl = __shfl_up_sync(kFull, lincl, 1);
    if (lane == 0) lexcl = 0.0;
    const unsigned cross = __ballot_sync(kFull, lsum > 0.0 && lincl > target);
    const unsigned pos = __ballot_sync(kFull, lsum > 0.0);
    // the crossing lane, else (rounding corner) the last lane with mass
    const int ln = cross ? __ffs(cross) - 1 : (pos ? 31 - __clz(pos) : 0);
    int mine = -1, last = -1;
    double mbase = 0.0, lbase = 0.0;
    if (lane == ln) {
      double cum = lexcl;
      for (int s0 = s_lo; s0 < s_hi; ++s0) {
        const double ms = mass_of(s0);
        if (ms > 0.0) {
          if (cross && cum + ms > target) {
            mine = s0;
            mbase = cum;
            break;
          }
          last = s0;
          lbase = cum;
        }
        cum += ms;
      }
    }
    us = __shfl_sync(kFull, mine, ln);
    base = __shfl_sync(kFull, mbase, ln);
    if (us < 0) {
      us = __shfl_sync(kFull, last, ln);
      base = __shfl_sync(kFull, lbase, ln);
      fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
    }
  }
  TAIL_STAMP(4);
  const double f = scale_of(us);
  uint4 rt[NV], rd[NV];
  load_sub_raw<T>(tp, a.V, us, rt);
  if (resid) load_sub_raw<T>(reinterpret_cast<const T*>(a.dl) + r.drow * a.ld_d, a.V, us, rd);
  const DrawRef DR = draw_ref<T>(rt, resid, r.M, (float)r.C, r.lam);
  int tok = -1, last_pos = -1;
  double lo = 0.0, hi = 0.0, lp_lo = 0.0, lp_hi = 0.0, vbase = base;
  // not unrolled: this runs once per sequence, so its instructions are cold;
  // a rolled loop re-fetches one vector's code from the instruction cache
  // instead of NV copies from L2 (ncu: the per-CTA code of k_tail stalled on
  // instruction fetch ~47% of its samples)
#pragma unroll 1
  for (int v = 0; v < NV; ++v) {
    float wv[VEC];
    vec_weights<T>(rt[v], rd[v], DR, wv);
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += wv[e];
    const double incl = wscan_d((double)ls, lane);
    const double pre = vbase + f * (incl - (double)ls);
    int cand = -1, lpos = -1;
    double clo = 0.0, chi = 0.0, llo = 0.0, lhi = 0.0;
    float run = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float before = run;
      run += wv[e];
      const double cb = pre + f * (double)before, ca = pre + f * (double)run;
      if (cand < 0 && wv[e] > 0.f && ca > target) {
        cand = e;
        clo = cb;
        chi = ca;
      }
      if (wv[e] > 0.f) {
        lpos = e;
        llo = cb;
        lhi = ca;
      }
    }
    const int tok_base = us * SUB + v * 32 * VEC;
    const unsigned bc = __ballot_sync(kFull, cand >= 0);
    if (bc) {
      const int lc = __ffs(bc) - 1;
      tok = tok_base + lc * VEC + __shfl_sync(kFull, cand, lc);
      lo = __shfl_sync(kFull, clo, lc);
      hi = __shfl_sync(kFull, chi, lc);
      break;
    }
    // remember the last positive-weight token for the rounding corner
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

template <typename T>
__global__ void __launch_bounds__(128) k_select(SelArgs a) {
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (i >= a.B) return;
  const SeqRec r = a.rec[i];
  select_seq<T>(a, i, r, SelSrcGlobal{a.smass + (long long)i * a.nsub, a.sref + (long long)i * a.nsub});
}

// ---------------------------------------------------------------------------
// k_tail: a2-a4 fused, one CTA (kFinThreads) per sequence: finalize (warp per
// position), then every warp forms the draw-weight masses of its slices of the
// drawn row (a4 first pass), then warp 0 selects the token. The drawn row is
// read by the CTA that decided it, so no launch boundary separates the steps.
// ---------------------------------------------------------------------------
// Extra arguments of the fused whole-step launch (dsde_step): the signal of
// every sequence (a5-a6) runs on the CTA's last warp as soon as its KLDs and
// a_i exist, and the CTA that finishes last computes the batch cap and next SLs
// (a7, single GPU; `counter` is zero before the launch and reset by that CTA).
struct StepExtra {
  SignalArgs sig;
  CapArgs cap;
  int fuse_cap;
  unsigned* counter;
};


// draw slices per row whose records k_tail keeps in shared memory (V <= 262144
// bf16 / 131072 fp32; larger vocabularies use the workspace)
constexpr int kTailMaxSub = 256;

template <typename T, bool STEP, int NW>
__global__ void __launch_bounds__(NW * 32, 1024 / (NW * 32)) k_tail(FinArgs fa, DrawArgs da, SelArgs sa,
                                                                   StepExtra sx) {
  constexpr int NVD = Traits<T>::NVD;
  __shared__ SeqRec s_rec;
  __shared__ double s_mass[kTailMaxSub], s_scale[kTailMaxSub];
  __shared__ float s_ref[kTailMaxSub];
  const int i = blockIdx.x;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_rec.mode = MODE_NONE;
  FinPre pre;
  if (warp == 0) pre = fin_prefetch<T>(fa, i);
  // programmatic dependent launch: the CTA may be resident before the stream
  // kernel has finished; wait for its completion (and memory) here
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  TAIL_STAMP(0);
  finalize_seq<T>(fa, i, &s_rec, &pre);
  __syncthreads();
  TAIL_STAMP(1);
  const SeqRec r = s_rec;
  const bool draw = r.mode == MODE_RESIDUAL || r.mode == MODE_BONUS || r.mode == MODE_ARGMAX;
#if DSDE_TAIL_TRACE
  unsigned smid;
  asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
  tail_stamp(5, ((unsigned long long)smid << 8) | (unsigned)r.mode);
#endif
  if (STEP && warp == NW - 1) {
    signal_seq(sx.sig, i);
    if (sx.fuse_cap) {
      // release ticket: this warp's sl_hat / state writes before the count; the
      // warp drawing the last ticket acquires and applies the cap (a7), without
      // waiting for any CTA's draw or select
      __syncwarp();
      unsigned old = 0;
      if ((threadIdx.x & 31) == 0)
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(sx.counter) : "memory");
      if (__shfl_sync(kFull, old, 0) == gridDim.x - 1) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        cap_warp(sx.cap);
        if ((threadIdx.x & 31) == 0) *sx.counter = 0u;
      }
    }
  }
  // slice records in shared memory when they fit (the select then reads no
  // global memory but the crossing slice), else in the workspace
  const bool smem = da.nsub <= kTailMaxSub;
  const long long q0 = (long long)i * da.nsub;
  if (draw) {
    for (int u = warp; u < da.nsub; u += NW) {
      uint4 rt[NVD], rd[NVD];
      const DrawUnit d = draw_unit_load<T>(da, u, r, rt, rd);
      if (smem) draw_unit_finish<T>(s_mass + u, s_ref + u, d, rt, rd);
      else draw_unit_finish<T>(da.smass + q0 + u, da.sref + q0 + u, d, rt, rd);
    }
  }
  __syncthreads();
  TAIL_STAMP(2);
  if (!draw) return;
  if (!smem) {
    if (warp == 0) select_seq<T>(sa, i, r, SelSrcGlobal{da.smass + q0, da.sref + q0});
    TAIL_STAMP(3);
    return;
  }
  if (r.mode == MODE_BONUS) {
    // the whole CTA rescales the bonus slice masses to the row max Mg (one fp64
    // exp per slice, in parallel), as select_seq would slice by slice
    __shared__ float s_wmax[NW];
    float mg = -INFINITY;
    for (int u = threadIdx.x; u < da.nsub; u += NW * 32) mg = max_nan(mg, s_ref[u]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mg = max_nan(mg, __shfl_xor_sync(kFull, mg, o));
    if ((threadIdx.x & 31) == 0) s_wmax[warp] = mg;
    __syncthreads();
    float Mg = s_wmax[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) Mg = max_nan(Mg, s_wmax[w]);
    for (int u = threadIdx.x; u < da.nsub; u += NW * 32) {
      const float ms = s_ref[u];
      const double f = ms == -INFINITY ? 0.0 : exp((double)ms - (double)Mg);
      s_scale[u] = f;
      s_mass[u] = f * s_mass[u];
    }
    __syncthreads();
  }
  if (warp == 0) select_seq<T>(sa, i, r, SelSrcSmem{s_mass, s_ref, s_scale});
  TAIL_STAMP(3);
}
