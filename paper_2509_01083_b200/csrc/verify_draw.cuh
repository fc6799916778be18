// verify_draw.cuh — a2-a4 of the verification pass after the row stream
// (included by verify.cu inside namespace dsde; uses its helpers). The same
// device functions serve k_tail (tail.cuh, the path of dsde_verify /
// dsde_step) and the staged kernels of the vocab-parallel path (vocab.cuh),
// so both give bit-identical results:
//
//   row_finalize  one warp per draft row: fp64 merge of the row's slice
//                 partials, KL(p||q), log p(x)/q(x) and the Philox accept test
//                 of its position (a2) -> a RowRes record;
//   seq_layout    one warp per sequence (lane j = position j): the first
//                 rejection a_i, the emitted-token layout and the draw record
//                 of the residual row a_i or the bonus row k_i (a3);
//   draw_mass     one warp per (sequence, vocab slice): the draw-weight mass of
//                 the slice of the drawn row (a4, first pass);
//   select_seq    one warp per sequence: the inverse CDF over the slice masses,
//                 then inside the crossing slice in ascending token order (a4,
//                 D7).

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
  int greedy;    // T = 0: accept iff x = argmax t, emit the argmax
  int dev_rows;  // dsde_config.device_rows: total is a capacity, sum k_i = cu_sl[B]
  float* ent;    // [sum k_i] optional out: draft entropy H(q) per row; partials carry Sd, E
  int v0;        // vocabulary offset of the rows (vocab-parallel shard; 0 otherwise)
  const float* temps;  // [B] per-sequence temperature (D20) or NULL; T = 0: greedy for that sequence
  int masked;          // dsde_config.masked: -inf logits allowed (D21); partials carry Fm (sign: cc), Fa
  // vocab-parallel: the gathered partials are shard blocks
  // [nshards][total][ns_sh]; slice c of row r is block c / ns_sh, entry
  // r ns_sh + c % ns_sh (ns_sh = nsub, single block, when not sharded); the
  // accept-test logits t_x, d_x come from xlog[r] (gathered from the owner shard)
  int ns_sh;
  long long blk;
  const float2* xlog;
};

// Slice c of row r's partials (the sharded view of FinArgs).
struct PartView {
  const SubPartial* base;  // part + r ns_sh
  int ns_sh;
  long long blk;
  __device__ __forceinline__ const SubPartial* at(int c) const {
    if (c < ns_sh) return base + c;  // the first (unsharded: the only) block
    const int s = c / ns_sh;
    return base + (long long)s * blk + (c - s * ns_sh);
  }
};

// Sequence i verifies greedily (T = 0): the global mode or its temperature 0.
__device__ __forceinline__ bool seq_greedy(const FinArgs& a, int i) {
  return a.greedy || (a.temps && __ldg(a.temps + i) == 0.f);
}

// Per-row result of row_finalize (64 bytes).
struct RowRes {
  double kl;   // KL(p || q)
  double lam;  // log1p(y) = log sum_v p_v exp(-w_v)
  double C;    // reference t - d (an fp32 value)
  double S;    // sum_v exp(t_v - M)
  float M;     // reference max of t
  int amax;    // greedy: argmax of t (smallest index)
  int bits;    // RR_* bits
  int x;       // the draft token of the row
  double pad2[2];
};
static_assert(sizeof(RowRes) == 64, "RowRes layout");
enum { RR_FINITE = 1, RR_ACCEPT = 2, RR_NEAR = 4, RR_BADTOK = 8 };

// Sequence i's row range and whether it is well formed: 1 <= k_i <= DSDE_MAX_SL,
// rows inside the launch (and, unless device_rows, the last sequence ends at
// total). `ok_rows` distinguishes DSDE_DERR_ROWS from DSDE_DERR_BAD_SL.
__device__ __forceinline__ bool seq_ok(const FinArgs& a, int i, int& c0, int& k, bool* ok_rows = nullptr) {
  c0 = __ldg(a.cu_sl + i);
  const int c1 = __ldg(a.cu_sl + i + 1);
  k = c1 - c0;
  const bool range_ok = c0 >= 0 && k >= 1 && k <= DSDE_MAX_SL && c1 <= a.total;
  const bool rows_ok = a.dev_rows || (i != a.B - 1) || (c1 == a.total);
  if (ok_rows) *ok_rows = rows_ok;
  return range_ok && rows_ok;
}

// ---------------------------------------------------------------------------
// a2: fp64 merge of row r's slice partials (lanes over slices c) about the
// row's references. A slice's e_v = 2^(t_v L2s - ML2_c) with ML2_c =
// fl32(M_c log2 e), the product the stream kernel rounded (SumRef), so its
// sums are exactly about M'_c = ML2_c ln 2 (not M_c): the merge uses M'_c
// (s = e^(M'_c - M'), M' = the largest). With Delta = C_c - C (C = fp32(M -
// max d)) and E1 = s e^-Delta:
//   S += s S_c,  A += s (A_c + S_c Delta),
//   D += E1 D_c - A_c s expm1(-Delta) + S_c s g(Delta),  g(x) = expm1(-x) + x.
// f = e e^-w of a slice lives in the frame M'_c - C_c, so its sums (ENT: Sd,
// E; MASK: Fp) are carried over with E1 (E shifted by ln E1); MASK's Fm is
// about fl32(maxd_c log2 e) ln 2 and is carried into the row's f frame.
// Partials are read with ld.global.cg: other SMs wrote them. Result in every
// lane.
// ---------------------------------------------------------------------------
struct RowSums {
  double S, A, D, Sd, E;  // ENT: Sd, E (draft entropy sums); MASK: Sd = Fm, E = Fp (row f frame)
  float M, Dmax;
  int cc;                 // MASK: some token the draft masks has p > 0
};

__device__ __forceinline__ double ref_nats(float m) {  // the stream's reference of a max m: fl32(m log2 e) ln 2
  return (double)__fmul_rn(m, kLog2e) * kLn2d;
}

__device__ __forceinline__ RowSums row_merge(const PartView P, int nc, bool ent, bool mask = false) {
  const int lane = threadIdx.x & 31;
  float Ml = -INFINITY, Dl = -INFINITY;
  for (int c = lane; c < nc; c += 32) {
    Ml = max_nan(Ml, __ldcg(&P.at(c)->M));
    Dl = fmaxf(Dl, __ldcg(&P.at(c)->maxd));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Ml = max_nan(Ml, __shfl_xor_sync(kFull, Ml, o));
    Dl = fmaxf(Dl, __shfl_xor_sync(kFull, Dl, o));
  }
  const double Mr = ref_nats(Ml), C = (double)(Ml - Dl);  // C is an fp32 value
  double S = 0.0, A = 0.0, D = 0.0, Sd = 0.0, E = 0.0;
  int cc = 0;
  for (int c = lane; c < nc; c += 32) {
    const float4 q0 = __ldcg(reinterpret_cast<const float4*>(P.at(c)));
    const float4 q1 = __ldcg(reinterpret_cast<const float4*>(P.at(c)) + 1);
    const double qS = q0.x, qA = q0.y, qD = q0.z, qC = q1.x;
    if (mask) {
      // Fm about the slice's fl32(maxd log2 e) ln 2, into the row's f frame Mr - C
      Sd += exp(ref_nats(q1.y) - (Mr - C)) * fabs((double)q1.z);
      cc |= signbit(q1.z) ? 1 : 0;
      if (q0.w == -INFINITY) continue;  // a slice whose target logits are all masked: only Fm
    }
    const double ls = ref_nats(q0.w) - Mr;
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
    if (ent && q1.z > 0.f) {
      // the draft's sums in the row's f frame: Sd += E1 Sd_c, E += E1 (E_c + ln(E1) Sd_c)
      Sd += E1 * (double)q1.z;
      E += E1 * ((double)q1.w + (ls - dl) * (double)q1.z);
    }
    if (mask) E += E1 * (double)q1.w;  // Fp
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_xor_sync(kFull, S, o);
    A += __shfl_xor_sync(kFull, A, o);
    D += __shfl_xor_sync(kFull, D, o);
  }
  if (ent || mask) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Sd += __shfl_xor_sync(kFull, Sd, o);
      E += __shfl_xor_sync(kFull, E, o);
    }
  }
  if (mask) cc = __any_sync(kFull, cc);
  return RowSums{S, A, D, Sd, E, Ml, Dl, cc};
}

// Greedy (T = 0): row argmax of t, smallest index among equal maxima (D18): the
// first slice holding the row max (slices are in token order), re-read vector
// by vector (token order is vector-major) until a lane holds the max.
template <typename T>
__device__ __forceinline__ int row_argmax(const FinArgs& a, const PartView P, int nc, float Ml,
                                          const T* trow) {
  constexpr int VEC = Traits<T>::VEC, SUB = sub_elems<T>();
  const int lane = threadIdx.x & 31;
  unsigned cs = 0x7fffffffu;
  for (int c = lane; c < nc; c += 32)
    if (__ldcg(&P.at(c)->M) == Ml) cs = min(cs, (unsigned)c);
  cs = __reduce_min_sync(kFull, cs);
  int amax = 0x7fffffff;
  if (cs < (unsigned)nc) {
    const T* row = trow + cs * SUB;
    const int left = a.V - (int)cs * SUB;
    for (int v = 0; v * 32 * VEC < min(SUB, left); ++v) {
      const int e0 = (v * 32 + lane) * VEC;
      int first = 0x7fffffff;
#pragma unroll
      for (int e = VEC - 1; e >= 0; --e)
        if (e0 + e < left && load_logit<T>(row + e0 + e) == Ml) first = e0 + e;
      const unsigned hit = __ballot_sync(kFull, first != 0x7fffffff);
      if (hit) {
        amax = a.v0 + (int)cs * SUB + __shfl_sync(kFull, first, __ffs(hit) - 1);
        break;
      }
    }
  }
  return amax;
}

// The accept-test inputs of draft row r = cu_sl[i] + j (lane 0): the token x,
// t_x, d_x and the Philox uniform of slot cu_sl[i] + i + j. They depend only
// on the step's inputs, so k_tail gathers them before griddepcontrol.wait,
// while the stream kernel still runs.
struct RowPre {
  int x;
  float tx, dx;
  double uacc, usmp;
};

template <typename T>
__device__ __forceinline__ RowPre row_prefetch(const FinArgs& a, int r, int i) {
  RowPre p{0, 0.f, 0.f, 0.0, 0.0};
  if ((threadIdx.x & 31) == 0) {
    const long long slot = (long long)r + i;
    p.x = __ldg(a.tokens + r);
    if (a.xlog) {  // vocab-parallel: the owner shard's t_x, d_x
      const float2 g = __ldcg(a.xlog + r);
      p.tx = g.x;
      p.dx = g.y;
    } else if (p.x >= 0 && p.x < a.V) {
      p.tx = load_logit<T>(reinterpret_cast<const T*>(a.tl) + slot * a.ld_t + p.x);
      p.dx = load_logit<T>(reinterpret_cast<const T*>(a.dl) + (long long)r * a.ld_d + p.x);
    }
    if (!seq_greedy(a, i)) {
      const Uniforms U = philox_uniforms(__ldg(a.seeds + slot));
      p.uacc = U.acc;
      p.usmp = U.smp;  // the recovery draw's uniform if this position is the first rejection
    }
  }
  return p;
}

// a2 for draft row r = cu_sl[i] + j (one warp); pre: the row's row_prefetch,
// or nullptr to gather it here (its latency then overlaps the merge). Returns
// the record in every lane.
template <typename T>
__device__ __forceinline__ RowRes row_finalize(const FinArgs& a, int r, int i, const RowPre* pre = nullptr) {
  const int lane = threadIdx.x & 31;
  const long long slot = (long long)r + i;
  const T* trow = reinterpret_cast<const T*>(a.tl) + slot * a.ld_t;
  const RowPre in = pre ? *pre : row_prefetch<T>(a, r, i);
  const int x = in.x;
  const float tx = in.tx, dx = in.dx;
  const double uacc = in.uacc;
  const double usmp = __shfl_sync(kFull, in.usmp, 0);
  const PartView P{a.part + (long long)r * a.ns_sh, a.ns_sh, a.blk};
  const bool greedy = seq_greedy(a, i);
  const RowSums R = row_merge(P, a.nsub, a.ent != nullptr, a.masked != 0);
  int amax = 0;
  if (greedy) amax = row_argmax<T>(a, P, a.nsub, R.M, trow);
  RowRes rr;
  rr.x = __shfl_sync(kFull, x, 0);
  rr.pad2[0] = usmp;  // u_smp of the row's slot (D6)
  rr.pad2[1] = 0.0;
  rr.amax = amax;
  rr.M = R.M;
  rr.C = (double)(R.M - R.Dmax);
  rr.S = R.S;
  // y = E_p[exp(-w)] - 1. KL = D/S + (log1p(y) - y) has no cancellation for
  // small KL; when y > 1 (the draft puts far more mass away from the
  // reference, e.g. disjoint supports) the equal form A/S + log1p(y) is used.
  // Masked logits (D21): in the row's f frame, Fp = sum_{supp p} e e^-w (the
  // draft mass on supp p; = (1 + y) S without masks) and Fm = the draft mass on
  // the tokens the target masks. q's normaliser is Fp + Fm, so log p/q at x and
  // the residual use lam' = log((Fp + Fm) / S) = log1p(y) - log Q with
  // Q = Fp / (Fp + Fm), and KL = (the formula) - log Q. When the draft masks a
  // token of supp p (cc), KL = +inf and y (which then omits that mass) is not
  // used: lam' = log(Fp / S) - log Q.
  const double y = (R.D - R.A) / R.S;
  const double lam = log1p(y);
  const bool kl_inf = a.masked && R.cc;
  const double lq = a.masked ? log1p(R.Sd / R.E) : 0.0;  // -log Q >= 0
  rr.lam = kl_inf ? log(R.E / R.S) + lq : lam + lq;
  rr.kl = kl_inf ? (double)INFINITY : fmax(0.0, (y <= 1.0 ? R.D / R.S + (lam - y) : R.A / R.S + lam) + lq);
  bool fin = isfinite(R.S) && isfinite(R.A) && isfinite(R.D) && R.S > 0.0 && isfinite((double)R.M) &&
             isfinite(rr.C) && (kl_inf || isfinite(rr.kl)) && isfinite(rr.lam);
  int bits = 0;
  if (lane == 0) {
    if (a.ent) a.ent[r] = (float)(log(R.Sd) - R.E / R.Sd);  // H(q) = log Sd - E / Sd (E <= 0)
    if (x < 0 || x >= a.V) {
      bits |= RR_BADTOK;
    } else {
      const float invT = inv_temp(a.temps, i);
      // log p(x) - log q(x) at the sequence's temperature
      const double lr = ((double)tx - (double)dx) * (double)invT - rr.C + rr.lam;
      if (a.masked && dx == -INFINITY) bits |= RR_BADTOK;  // q(x) = 0: x cannot have been drafted
      fin = fin && (isfinite(lr) || (a.masked && lr == -INFINITY));  // p(x) = 0: a certain rejection
      if (greedy) {
        if (x == amax) bits |= RR_ACCEPT;  // T = 0: the draft token must be the target argmax
      } else {
        const double pacc = lr >= 0.0 ? 1.0 : exp(lr);
        if (uacc < pacc) bits |= RR_ACCEPT;
        if (fabs(uacc - pacc) < 1e-6) bits |= RR_NEAR;
      }
    }
    if (a.temps) {
      const float Ti = __ldg(a.temps + i);
      if (!(Ti >= 0.f && Ti < INFINITY)) fin = false;  // a negative / non-finite temperature
    }
    if (fin) bits |= RR_FINITE;
  }
  rr.bits = __shfl_sync(kFull, bits, 0);
  return rr;
}

__device__ __forceinline__ void store_rowres(RowRes* dst, const RowRes& r) {
  if ((threadIdx.x & 31) == 0) *dst = r;
}

__device__ __forceinline__ RowRes load_rowres(const RowRes* p) {
  RowRes r;
  const double2 a0 = __ldcg(reinterpret_cast<const double2*>(p));
  const double2 a1 = __ldcg(reinterpret_cast<const double2*>(p) + 1);
  const int4 b = __ldcg(reinterpret_cast<const int4*>(p) + 2);
  r.kl = a0.x;
  r.lam = a0.y;
  r.C = a1.x;
  r.S = a1.y;
  r.M = __int_as_float(b.x);
  r.amax = b.y;
  r.bits = b.z;
  r.x = b.w;
  const double2 c = __ldcg(reinterpret_cast<const double2*>(p) + 3);
  r.pad2[0] = c.x;
  r.pad2[1] = c.y;
  return r;
}

// Outputs of a sequence with a data error: accepted_len -1, all-pad tokens, NaN KLD.
__device__ __forceinline__ void seq_error_outputs(const FinArgs& a, int i, int c0, int k, int code) {
  const int lane = threadIdx.x & 31;
  const long long slot0 = (long long)c0 + i;
  for (int j = lane; j < k; j += 32) a.kld[c0 + j] = NAN;
  for (int j = lane; j <= k; j += 32) {
    a.emitted[slot0 + j] = DSDE_PAD;
    if (a.flags) a.flags[slot0 + j] = 0;
  }
  if (lane == 0) {
    a.acc_len[i] = -1;
    raise_device_error(a.err, code, i);
  }
}

__device__ __forceinline__ SeqRec error_rec(long long slot0) {
  SeqRec r;
  r.mode = MODE_ERROR;
  r.slot = (int)slot0;
  r.trow = slot0;
  r.drow = -1;
  r.M = 0.f;
  r.invT = 1.f;
  r.C = r.lam = r.u = r.S = 0.0;
  return r;
}

// a3 (one warp; lane j < k holds position j's RowRes): the first rejection a_i,
// KLDs, the emitted-token layout (x_0 .. x_{a-1}, the drawn token at a, pads
// after), flags and the draw record (written by lane a to *out).
// Returns a_i (-1 on a data error) in every lane. u_bonus: the bonus slot's
// u_smp when the caller gathered it (k_tail, before griddepcontrol.wait), else
// NULL.
__device__ __forceinline__ int seq_layout(const FinArgs& a, int i, int c0, int k, const RowRes& rr,
                                          SeqRec* out, const double* u_bonus = nullptr) {
  const int lane = threadIdx.x & 31;
  const long long slot0 = (long long)c0 + i;
  const unsigned bt = __ballot_sync(kFull, lane < k && (rr.bits & RR_BADTOK));
  const unsigned nf = __ballot_sync(kFull, lane < k && !(rr.bits & RR_FINITE));
  const unsigned am = __ballot_sync(kFull, lane < k && (rr.bits & RR_ACCEPT));
  if (bt | nf) {
    seq_error_outputs(a, i, c0, k, bt ? DSDE_DERR_BAD_TOKEN : DSDE_DERR_NONFINITE);
    if (lane == 0) *out = error_rec(slot0);
    return -1;
  }
  const int acc_run = __ffs(~am) - 1;  // first rejected lane (lanes >= k never accept)
  const int aa = acc_run < k ? acc_run : k;
  if (lane < k) a.kld[c0 + lane] = (float)rr.kl;
  if (lane <= k) {
    a.emitted[slot0 + lane] = lane < aa ? rr.x : DSDE_PAD;
    if (a.flags)
      a.flags[slot0 + lane] = ((rr.bits & RR_NEAR) && lane <= aa && lane < k) ? DSDE_FLAG_ACCEPT_NEAR_TIE : 0;
  }
  if (lane == 0) a.acc_len[i] = aa;
  if (lane == aa) {
    const bool greedy = seq_greedy(a, i);
    SeqRec r;
    r.invT = greedy ? 1.f : inv_temp(a.temps, i);
    r.S = 0.0;
    r.slot = (int)(slot0 + aa);
    r.trow = slot0 + aa;
    r.drow = -1;
    r.M = 0.f;
    r.C = r.lam = r.u = 0.0;
    if (greedy) {
      // T = 0: the recovery token is the argmax of row aa (known from its
      // finalize); the bonus row's argmax is found by the draw pass
      if (aa < k) {
        a.emitted[slot0 + aa] = rr.amax;
        r.mode = MODE_NONE;
      } else {
        r.mode = MODE_ARGMAX;
      }
    } else {
      // the recovery draw's u_smp was gathered with the row (RowRes.pad2[0]);
      // the bonus slot has no row
      r.u = aa < k ? rr.pad2[0] : u_bonus ? *u_bonus : philox_uniforms(__ldg(a.seeds + slot0 + aa)).smp;
      if (aa < k) {
        r.mode = MODE_RESIDUAL;
        r.drow = (long long)c0 + aa;
        r.M = rr.M;
        r.C = rr.C;
        r.lam = rr.lam;
        r.S = rr.S;
      } else {
        r.mode = MODE_BONUS;
      }
    }
    *out = r;
  }
  return aa;
}

// ---------------------------------------------------------------------------
// Draw weights of one lane over the slice u of a row (NV 16-byte vectors per
// lane, token u*SUB + (v*32 + lane)*VEC + e), from raw words; the reference
// (residual: M of the row; bonus: warp max of t over the slice):
//   residual: rho_v = e_v (1 - exp(-z_v)) for z_v > 0, else 0, with
//             e_v = exp(t_v - M), z_v = w_v + lam, w_v = (t_v - d_v) - C exact,
//             lam added as hi + lo floats; 1 - exp(-z) = z (1 - z h(-z)) for
//             |z| < 1/2 (no cancellation), 1 - 2^(-z log2 e) otherwise;
//   bonus:    p_v up to a scale: exp(t_v - m_u) about the slice max m_u,
//             rescaled by exp(m_u - max_u m_u) in fp64 by the select.
// The select recomputes every weight bit-identically from the same words.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ float2 resid_pair_exact(float2 tt, float2 dd, float2 nML2, float khi, float klo,
                                                   float invT) {
  const float l2 = kLog2e * invT;
  const float2 L2 = make_float2(l2, l2), nL2 = make_float2(-kLog2e, -kLog2e);
  const float2 ONE = make_float2(1.f, 1.f);
  // degree 5 on |z| <= 1/2 (1.1e-7 relative; tools/fit_g.py --deg 5 --range 0.5)
  const float2 K5 = make_float2(-1.9962186343036592e-04f, -1.9962186343036592e-04f);
  const float2 K4 = make_float2(1.3982197269797325e-03f, 1.3982197269797325e-03f);
  const float2 K3 = make_float2(-8.333181962370872e-03f, -8.333181962370872e-03f);
  const float2 K2 = make_float2(4.166579246520996e-02f, 4.166579246520996e-02f);
  const float2 K1 = make_float2(-1.666666716337204e-01f, -1.666666716337204e-01f);
  const float2 K0 = make_float2(0.5f, 0.5f);
  const float2 xt = __ffma2_rn(tt, L2, nML2);
  const float2 ev = make_float2(fast_exp2(xt.x), fast_exp2(xt.y));  // 0 for padding
  // z = (t - d) / T - (C - lam), the constant carried as khi + klo
  float2 z = diff2<T>(tt, dd, khi, invT);  // t - d exact (bf16) or TwoDiff (fp32)
  z = __fadd2_rn(z, make_float2(-klo, -klo));
  float2 pz = __ffma2_rn(K5, z, K4);
  pz = __ffma2_rn(pz, z, K3);
  pz = __ffma2_rn(pz, z, K2);
  pz = __ffma2_rn(pz, z, K1);
  pz = __ffma2_rn(pz, z, K0);
  const float2 sm = __fmul2_rn(z, __ffma2_rn(make_float2(-z.x, -z.y), pz, ONE));  // z (1 - z h(-z))
  const float2 xz = __fmul2_rn(z, nL2);
  const float2 bg = __fadd2_rn(ONE, make_float2(-fast_exp2(xz.x), -fast_exp2(xz.y)));  // 1 - e^-z
  // 1 - e^-z <= 0 for z <= 0 in both forms (the polynomial only on |z| < 1/2;
  // beyond, 1 - 2^(-z log2 e) has a relative error below ~3.4e-7), so
  // max(0, .) zeroes exactly the tokens with p_v <= q_v (fmaxf drops the NaN
  // of padding, 0 * -inf)
  const float2 om = make_float2(fabsf(z.x) < 0.5f ? sm.x : bg.x, fabsf(z.y) < 0.5f ? sm.y : bg.y);
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
  float M, khi, klo;  // residual: row reference M (of t / T), C - lam = khi + klo
  float m;            // bonus: the slice's warp max of t (raw; the reference is m / T)
  float invT;         // 1 / T (D20)
};

// Warp-wide max of t over a lane's N vectors (NaN-propagating; packed
// max.NaN.bf16x2 for bf16: max is exact, so any grouping gives the same value).
template <typename T, int N>
__device__ __forceinline__ float lane_tmax(const uint4 (&rt)[N], float m) {
  if constexpr (sizeof(T) == 2) {
    __nv_bfloat162 b0 = __floats2bfloat162_rn(-INFINITY, -INFINITY), b1 = b0;
#pragma unroll
    for (int v = 0; v < N; ++v) {
      const uint32_t w4[4] = {rt[v].x, rt[v].y, rt[v].z, rt[v].w};
      b0 = __hmax2_nan(b0, *reinterpret_cast<const __nv_bfloat162*>(&w4[0]));
      b1 = __hmax2_nan(b1, *reinterpret_cast<const __nv_bfloat162*>(&w4[1]));
      b0 = __hmax2_nan(b0, *reinterpret_cast<const __nv_bfloat162*>(&w4[2]));
      b1 = __hmax2_nan(b1, *reinterpret_cast<const __nv_bfloat162*>(&w4[3]));
    }
    const __nv_bfloat162 b = __hmax2_nan(b0, b1);
    return max_nan(m, max_nan(__low2float(b), __high2float(b)));
  } else {
#pragma unroll
    for (int v = 0; v < N; ++v) m = vec_tmax<T>(rt[v], m);
    return m;
  }
}

__device__ __forceinline__ float warp_max_nan(float m) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max_nan(m, __shfl_xor_sync(kFull, m, o));
  return m;
}

__device__ __forceinline__ DrawRef draw_ref(bool resid, float M, float Cf, double lam, float m, float invT) {
  DrawRef R;
  R.resid = resid;
  R.invT = invT;
  R.M = M;
  const double K = (double)Cf - lam;
  R.khi = (float)K;
  R.klo = (float)(K - (double)R.khi);
  R.m = m;
  return R;
}

// Draw weights of the VEC tokens of one lane vector.
template <typename T>
__device__ __forceinline__ void vec_weights(const uint4& t4, const uint4& d4, const DrawRef& R,
                                            float (&w)[Traits<T>::VEC]) {
  constexpr int VEC = Traits<T>::VEC;
  const uint4 rt[1] = {t4}, rd[1] = {d4};
  const float l2 = kLog2e * R.invT;
  const float2 L2 = make_float2(l2, l2);
  if (R.resid) {
    const float ML2 = R.M * kLog2e;
    const float2 nML2 = make_float2(-ML2, -ML2);
#pragma unroll
    for (int h = 0; h < VEC; h += 2) {
      const float2 r = resid_pair_exact<T>(pair_of<T>(rt, h), pair_of<T>(rd, h), nML2, R.khi, R.klo, R.invT);
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
  const float mL2 = R.m * l2;  // (t - m) / T in base 2
  const float2 nmL2 = make_float2(-mL2, -mL2);
#pragma unroll
  for (int h = 0; h < VEC; h += 2) {
    const float2 x = __ffma2_rn(pair_of<T>(rt, h), L2, nmL2);
    w[h] = fast_exp2(x.x);
    w[h + 1] = fast_exp2(x.y);
  }
}

// raw words of vectors [v0, v0 + N) of draw slice u of a row (draw / select
// passes): the non-coherent read-only path without L1 allocation (the logits
// are never written during a call; measured 2-8% faster tails than
// ld.global.cg: cfg3 64.7 -> 62.4 us, cfg4 112.7 -> 104.4 us)
template <typename T, int N>
__device__ __forceinline__ void load_vecs(const T* row, int V, int u, int v0, uint4 (&r)[N]) {
  constexpr int VEC = Traits<T>::VEC, SUB = draw_elems<T>();
  const int lane = threadIdx.x & 31;
  const T* base = row + u * SUB + (v0 * 32 + lane) * VEC;
  if (u * SUB + (v0 + N) * 32 * VEC <= V) {
    // every vector inside the row (all but the last slice): the N loads back
    // to back from one base address (a per-vector bounds branch makes the
    // compiler rebuild the 64-bit row address per vector: measured 35% slower
    // draws)
#pragma unroll
    for (int v = 0; v < N; ++v) r[v] = ld_stream_v4(base + v * 32 * VEC);
    return;
  }
#pragma unroll
  for (int v = 0; v < N; ++v) {
    const int e0 = u * SUB + ((v0 + v) * 32 + lane) * VEC;
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
// double per kept vector instead of one per vector), then lane 0 gathers them.
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
// a4 first pass, one warp: the draw-weight mass of draw slice u (1024 bf16 /
// 512 fp32 tokens: NVD vectors per lane, all loaded at once) of sequence i's
// drawn row (record r), written to mass_out / ref_out (lane 0). The mass is the
// per-vector fp32 lane sums summed over lanes in fp64 (warp_sum_vectors), in
// the select pass's grouping. Greedy bonus rows (ARGMAX) record the slice max
// of t and its first index instead.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void draw_mass_loaded(const SeqRec& r, const uint4 (&rt)[Traits<T>::NVD],
                                                 const uint4 (&rd)[Traits<T>::NVD], double* mass_out, float* ref_out) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NVD;
  const int lane = threadIdx.x & 31;
  const int mode = r.mode;
  DrawRef R;
  if (mode != MODE_RESIDUAL) {
    // bonus / argmax: the slice max of t first (the reference of the weights)
    const float m = warp_max_nan(lane_tmax<T, NV>(rt, -INFINITY));
    if (mode == MODE_ARGMAX) {
      int best = 0x7fffffff;
#pragma unroll
      for (int v = NV - 1; v >= 0; --v) {
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
    R = draw_ref(false, 0.f, 0.f, 0.0, m, r.invT);
  } else {
    R = draw_ref(true, r.M, (float)r.C, r.lam, 0.f, r.invT);
  }
  double x[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    float w[VEC];
    vec_weights<T>(rt[v], R.resid ? rd[v] : rt[v], R, w);
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += w[e];
    x[v] = (double)ls;
  }
  const double tot = warp_sum_vectors<NV>(x);
  if (lane == 0) {
    *mass_out = tot;
    // bonus: the raw slice max m of t (the weights' reference is m / T; the
    // select rescales by fl32(m invT), which is monotone in m)
    *ref_out = R.resid ? R.M : (R.m <= -1e30f ? -INFINITY : R.m);
  }
}

template <typename T>
__device__ __forceinline__ void draw_mass(const SeqRec& r, int u, int V, const void* tl, long long ld_t,
                                          const void* dl, long long ld_d, double* mass_out, float* ref_out) {
  constexpr int NV = Traits<T>::NVD;
  const int mode = r.mode;
  if (mode != MODE_RESIDUAL && mode != MODE_BONUS && mode != MODE_ARGMAX) return;
  const T* tp = reinterpret_cast<const T*>(tl) + r.trow * ld_t;
  uint4 rt[NV], rd[NV];
  load_vecs<T, NV>(tp, V, u, 0, rt);
  if (mode == MODE_RESIDUAL) load_vecs<T, NV>(reinterpret_cast<const T*>(dl) + r.drow * ld_d, V, u, 0, rd);
  draw_mass_loaded<T>(r, rt, rd, mass_out, ref_out);
}

// Bonus / argmax rows read only t: two draw slices (u0, and u1 < nd when
// valid) per call with all their loads in flight at once (the per-warp loop is
// latency-bound on one slice's 4 vectors).
template <typename T>
__device__ __forceinline__ void draw_mass_t2(const SeqRec& r, int u0, int u1, int nd, int V, const void* tl,
                                             long long ld_t, double* m0, float* r0, double* m1, float* r1) {
  constexpr int NV = Traits<T>::NVD;
  const T* tp = reinterpret_cast<const T*>(tl) + r.trow * ld_t;
  uint4 a0[NV], a1[NV];
  load_vecs<T, NV>(tp, V, u0, 0, a0);
  if (u1 < nd) load_vecs<T, NV>(tp, V, u1, 0, a1);
  draw_mass_loaded<T>(r, a0, a0, m0, r0);
  if (u1 < nd) draw_mass_loaded<T>(r, a1, a1, m1, r1);
}

// ---------------------------------------------------------------------------
// a4 second pass, one warp: the inverse-CDF select of sequence i from its
// slice masses (mass[s], ref[s], s < nsub, read with ld.global.cg) — D7: the
// smallest token v with C_v > u R in ascending token order.
// ---------------------------------------------------------------------------
struct SelArgs {
  int B, V, nsub;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  int32_t* emitted;
  uint8_t* flags;
  int32_t* err;
  int v0;  // vocabulary offset of the rows (vocab-parallel shard)
  // vocab-parallel: this shard's draw slices [s_lo, s_lo + nd_sh)
  // of the row's nsub, its columns' V; tok_out != NULL: the selected token
  // (global id, sample flags << 24) or -1 when another shard owns the
  // crossing slice, instead of writing emitted / flags
  int s_lo, nd_sh, Vs;
  int32_t* tok_out;
};

#ifndef DSDE_TAIL_TRACE
#define DSDE_TAIL_TRACE 0
#endif

// Slice records: in global memory (ld.global.cg: written by other warps of the
// launch) or in the CTA's shared memory (SMEM; the bonus masses then already
// rescaled to the row max by the CTA, `sscale` holding the factors).
template <bool SMEM>
struct SliceSrc {
  const double* mass;
  const float* ref;
  const double* scale;  // SMEM only
  __device__ __forceinline__ double m(int s) const { return SMEM ? mass[s] : __ldcg(mass + s); }
  __device__ __forceinline__ float r(int s) const { return SMEM ? ref[s] : __ldcg(ref + s); }
};

template <typename T, bool SMEM = false, typename Src = SliceSrc<SMEM>>
__device__ __forceinline__ void select_seq(const SelArgs& a, int i, const SeqRec& r, const Src src) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NVD, SUB = draw_elems<T>();
  const int lane = threadIdx.x & 31;
  if (r.mode == MODE_ARGMAX) {
    // greedy bonus token: the smallest index among the slices holding the row max
    float Mg = -INFINITY;
    for (int s0 = lane; s0 < a.nsub; s0 += 32) Mg = max_nan(Mg, src.r(s0));
    Mg = warp_max_nan(Mg);
    unsigned cand = 0x7fffffffu;
    for (int s0 = lane; s0 < a.nsub; s0 += 32)
      if (src.r(s0) == Mg) cand = min(cand, (unsigned)(s0 * SUB + (int)src.m(s0)));
    cand = __reduce_min_sync(kFull, cand);
    if (lane == 0) {
      if (Mg != Mg || cand >= (unsigned)a.V) {
        a.emitted[r.slot] = DSDE_PAD;
        raise_device_error(a.err, DSDE_DERR_NONFINITE, i);
      } else {
        a.emitted[r.slot] = a.v0 + (int)cand;
      }
    }
    return;
  }
  if (r.mode != MODE_RESIDUAL && r.mode != MODE_BONUS) return;
  const bool resid = r.mode == MODE_RESIDUAL;
  const int nsub = a.nsub;
  float Mg = -INFINITY;  // bonus: the row's largest slice reference fl32(m invT)
  if (!resid && !SMEM) {
    for (int s0 = lane; s0 < nsub; s0 += 32) Mg = max_nan(Mg, src.r(s0));
    Mg = __fmul_rn(warp_max_nan(Mg), r.invT);
  }
  auto scale_of = [&](int s0) -> double {  // slice mass scale to the common reference
    if (resid) return 1.0;
    if (SMEM) return src.scale[s0];
    const float ms = src.r(s0);
    return ms == -INFINITY ? 0.0 : exp((double)__fmul_rn(ms, r.invT) - (double)Mg);
  };
  // shared-memory bonus masses are already rescaled
  auto mass_of = [&](int s0) -> double { return (SMEM || resid) ? src.m(s0) : scale_of(s0) * src.m(s0); };
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
    if (a.tok_out) {  // vocab-parallel: the D7 fallback scans a whole row; not supported
      if (lane == 0) {
        a.tok_out[i] = -2;
        raise_device_error(a.err, isfinite(R) ? DSDE_DERR_VP_FALLBACK : DSDE_DERR_NONFINITE, i);
      }
      return;
    }
    if (lane == 0) {
      // residual mass 0 (p <= q everywhere in fp32; D7 fallback: draw from p
      // of the same target row, one lane) or a non-finite bonus row
      if (resid && isfinite(R)) {
        double tot = 0.0;
        for (int v = 0; v < a.V; ++v) tot += exp((double)load_logit<T>(tp + v) * (double)r.invT - (double)r.M);
        const double target = r.u * tot;
        double cum = 0.0;
        int tok = 0;
        for (int v = 0; v < a.V; ++v) {
          const double wv = exp((double)load_logit<T>(tp + v) * (double)r.invT - (double)r.M);
          cum += wv;
          if (wv > 0.0) tok = v;
          if (wv > 0.0 && cum > target) break;
        }
        a.emitted[r.slot] = a.v0 + tok;
        if (a.flags) a.flags[r.slot] |= DSDE_FLAG_FALLBACK;
      } else {
        a.emitted[r.slot] = DSDE_PAD;
        raise_device_error(a.err, DSDE_DERR_NONFINITE, i);
      }
    }
    return;
  }
  const double target = r.u * R;
  // crossing slice: first s with prefix(s) > target (fallback: last with
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
  const double f = scale_of(us);
  // vocab-parallel: only the shard owning the crossing slice scans it (with
  // its own columns); the others report -1
  const int Vl = a.tok_out ? a.Vs : a.V;
  if (a.tok_out) {
    if (us < a.s_lo || us >= a.s_lo + a.nd_sh) {
      if (lane == 0) a.tok_out[i] = -1;
      return;
    }
    us -= a.s_lo;
  }
  const T* dp = resid ? reinterpret_cast<const T*>(a.dl) + r.drow * a.ld_d : tp;
  // the crossing slice's bonus reference: the raw slice max draw_mass
  // recorded (the record index under vocab parallelism is us + s_lo)
  const float m_raw = resid ? 0.f : src.r(a.tok_out ? us + a.s_lo : us);
  const DrawRef DR = draw_ref(resid, r.M, (float)r.C, r.lam, m_raw, r.invT);
  int tok = -1, last_pos = -1;
  double lo = 0.0, hi = 0.0, lp_lo = 0.0, lp_hi = 0.0, vbase = base;
  // one vector at a time, not unrolled: this runs once per sequence, so its
  // instructions are cold, and the kernel's 64-register budget is shared with
  // the draw loop (hoisting all the slice's loads spilled there: measured
  // slower draws and selects; an L1 prefetch of the slice: no gain)
#pragma unroll 1
  for (int v = 0; v < NV; ++v) {
    uint4 rt[1], rd[1];
    load_vecs<T, 1>(tp, Vl, us, v, rt);
    if (resid) load_vecs<T, 1>(dp, Vl, us, v, rd);
    else rd[0] = rt[0];
    float wv[VEC];
    vec_weights<T>(rt[0], rd[0], DR, wv);
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
  if (tok < 0) {  // rounding corner: u R within rounding of the slice total
    tok = last_pos;
    lo = lp_lo;
    hi = lp_hi;
    fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
  }
  if (lane == 0) {
    if (fabs(r.u - lo / R) < 1e-6 || fabs(r.u - hi / R) < 1e-6) fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
    if (a.tok_out) {
      a.tok_out[i] = (a.v0 + (tok < 0 ? 0 : tok)) | ((int)fl << 24);  // tokens < 2^24
    } else {
      a.emitted[r.slot] = a.v0 + (tok < 0 ? 0 : tok);
      if (a.flags) a.flags[r.slot] |= fl;
    }
  }
}

// ---------------------------------------------------------------------------
// D23 path: p's statistics per stream slice of one target row — the draft
// row's SubPartials (S at +0, M/T at +3: stride 8 floats, offset 3); written by
// the stream kernel, read with ld.global.cg.
// ---------------------------------------------------------------------------
struct PRow {
  const float* base;
  int stride, moff;
  __device__ __forceinline__ float S(int s) const { return __ldcg(base + (long long)s * stride); }
  __device__ __forceinline__ float M(int s) const { return __ldcg(base + (long long)s * stride + moff); }
};

struct PSel {
  int tok;     // -1: p's mass is not a finite positive number (non-finite row)
  uint8_t fl;  // DSDE_FLAG_SAMPLE_NEAR_TIE when u is within 1e-6 of the token's CDF edges
  float t;     // the token's logit (the proposal's accept test)
};

// lane vector v of stream slice u of a row (padding past V: weight exactly 0),
// through L1 (p_select prefetched the slice there)
template <typename T>
__device__ __forceinline__ uint4 load_svec(const T* row, int V, int u, int v) {
  constexpr int VEC = Traits<T>::VEC, SUB = sub_elems<T>();
  const int e0 = u * SUB + (v * 32 + (threadIdx.x & 31)) * VEC;
  if (e0 + VEC <= V) return __ldg(reinterpret_cast<const uint4*>(row + e0));
  T b[VEC];
#pragma unroll
  for (int e = 0; e < VEC; ++e) b[e] = (e0 + e < V) ? row[e0 + e] : pad_bits<T>();
  return *reinterpret_cast<const uint4*>(b);
}

// p's CDF over the stream slices of one row, shared by a CTA's warps: pre[s] =
// sum_{s' <= s} e^(M'_s' - M') S_s' in fp64 (slice order), ml2[s] =
// fl32(M_s/T log2 e) (the stream's exact base-2 reference, -inf: no mass),
// Mr = M' (nats) and P = pre[nsub - 1].
struct PCdf {
  double* pre;
  float* ml2;
  double Mr, P;
};

// One warp builds the PCdf of a row from its streamed slice statistics (lanes
// own contiguous slice spans; one fp64 warp scan). Returns P in every lane
// (not a finite positive number: a non-finite row).
__device__ __noinline__ double pcdf_build(const PRow src, int nsub, double* pre, float* ml2, double* Mr_out) {
  const int lane = threadIdx.x & 31;
  float Mg = -INFINITY;
  for (int s0 = lane; s0 < nsub; s0 += 32) Mg = max_nan(Mg, src.M(s0));
  Mg = warp_max_nan(Mg);
  const double Mr = ref_nats(Mg);
  const int cw = (nsub + 31) >> 5;
  const int s_lo = min(lane * cw, nsub), s_hi = min(s_lo + cw, nsub);
  double lsum = 0.0;
  for (int s0 = s_lo; s0 < s_hi; ++s0) {  // the masses (pre[] holds them until the scan)
    const float m = src.M(s0);
    const double ms = m != -INFINITY ? exp(ref_nats(m) - Mr) * (double)src.S(s0) : 0.0;
    pre[s0] = ms;
    ml2[s0] = m == -INFINITY ? -INFINITY : __fmul_rn(m, kLog2e);
    lsum += ms;
  }
  const double lincl = wscan_d(lsum, lane);
  double cum = lincl - lsum;
  for (int s0 = s_lo; s0 < s_hi; ++s0) {
    cum += pre[s0];
    pre[s0] = cum;
  }
  *Mr_out = Mg != Mg ? (double)NAN : Mr;
  return __shfl_sync(kFull, lincl, 31);
}

// One warp: p's inverse CDF (D7 applied to p, at the sequence's temperature)
// from a PCdf: the crossing slice (first s with mass and pre[s] > u P), its
// NV vectors prefetched at once, then per vector the weights
// e_v = 2^(t_v L2s - ml2[s]) (bit-identical to the stream's), an fp64 warp
// scan of the lane sums, and the smallest token with C_v > u P in ascending
// token order. Rounding
// corners (u P within rounding of a slice total) take the last positive-weight
// token and are flagged.
template <typename T>
__device__ __noinline__ PSel p_select(const PCdf c, int nsub, const T* trow, int V, float invT, double u) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, SUB = sub_elems<T>();
  const int lane = threadIdx.x & 31;
  PSel out{-1, 0, 0.f};
  const double P = c.P;
  if (!(P > 0.0) || !isfinite(P) || c.Mr != c.Mr) return out;
  const double target = u * P;
  int us = -1;
  for (int s0 = 0; s0 < nsub && us < 0; s0 += 32) {
    const int sl = s0 + lane;
    const double prev = sl == 0 ? 0.0 : sl < nsub ? c.pre[sl - 1] : 0.0;
    const bool cross = sl < nsub && c.pre[sl] > prev && c.pre[sl] > target;
    const unsigned b = __ballot_sync(kFull, cross);
    if (b) us = s0 + __ffs(b) - 1;
  }
  if (us < 0) {  // rounding corner: the last slice with mass
    out.fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
    for (int s0 = ((nsub - 1) & ~31); s0 >= 0 && us < 0; s0 -= 32) {
      const int sl = s0 + lane;
      const double prev = sl == 0 ? 0.0 : sl < nsub ? c.pre[sl - 1] : 0.0;
      const unsigned b = __ballot_sync(kFull, sl < nsub && c.pre[sl] > prev);
      if (b) us = s0 + 31 - __clz(b);
    }
    if (us < 0) return out;
  }
  const double base = us == 0 ? 0.0 : c.pre[us - 1];
  const float ML2 = c.ml2[us], l2 = __fmul_rn(kLog2e, invT);
  const double f = exp((double)ML2 * kLn2d - c.Mr);
  // the slice's NV vectors requested at once (into L1), then scanned one vector
  // at a time in a rolled loop: this code runs once per draw, cold, so its
  // size (instruction fetch) costs more than its arithmetic
  {
    const int e0 = us * SUB + (threadIdx.x & 31) * VEC;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (e0 + v * 32 * VEC + VEC <= V) asm volatile("prefetch.global.L1 [%0];" ::"l"(trow + e0 + v * 32 * VEC));
  }
  int tok = -1, last_pos = -1;
  double lo = 0.0, hi = 0.0, lp_lo = 0.0, lp_hi = 0.0, vbase = base;
  float tk = 0.f, lpt = 0.f;
#pragma unroll 1
  for (int v = 0; v < NV; ++v) {
    const uint4 xv[1] = {load_svec<T>(trow, V, us, v)};
    float wv[VEC], tv[VEC];
#pragma unroll
    for (int h = 0; h < VEC; h += 2) {
      const float2 tt = pair_of<T>(xv, h);
      tv[h] = tt.x;
      tv[h + 1] = tt.y;
      wv[h] = fast_exp2(__fmaf_rn(tt.x, l2, -ML2));
      wv[h + 1] = fast_exp2(__fmaf_rn(tt.y, l2, -ML2));
    }
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += wv[e];
    const double incl = wscan_d((double)ls, lane);
    const double pre = vbase + f * (incl - (double)ls);
    int cand = -1, lpos = -1;
    double clo = 0.0, chi = 0.0, llo = 0.0, lhi = 0.0;
    float ct = 0.f, lt = 0.f, run = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      const float before = run;
      run += wv[e];
      const double cb = pre + f * (double)before, ca = pre + f * (double)run;
      if (cand < 0 && wv[e] > 0.f && ca > target) {
        cand = e;
        clo = cb;
        chi = ca;
        ct = tv[e];
      }
      if (wv[e] > 0.f) {
        lpos = e;
        llo = cb;
        lhi = ca;
        lt = tv[e];
      }
    }
    const int tok_base = us * SUB + v * 32 * VEC;
    const unsigned bc = __ballot_sync(kFull, cand >= 0);
    if (bc) {
      const int lc = __ffs(bc) - 1;
      tok = tok_base + lc * VEC + __shfl_sync(kFull, cand, lc);
      lo = __shfl_sync(kFull, clo, lc);
      hi = __shfl_sync(kFull, chi, lc);
      tk = __shfl_sync(kFull, ct, lc);
      break;
    }
    const unsigned bp = __ballot_sync(kFull, lpos >= 0);
    if (bp) {
      const int lp = 31 - __clz(bp);
      last_pos = tok_base + lp * VEC + __shfl_sync(kFull, lpos, lp);
      lp_lo = __shfl_sync(kFull, llo, lp);
      lp_hi = __shfl_sync(kFull, lhi, lp);
      lpt = __shfl_sync(kFull, lt, lp);
    }
    vbase += f * __shfl_sync(kFull, incl, 31);
  }
  if (tok < 0) {  // rounding corner: u P within rounding of the slice total
    tok = last_pos;
    lo = lp_lo;
    hi = lp_hi;
    tk = lpt;
    out.fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
    if (tok < 0) return out;
  }
  out.tok = tok;
  out.t = tk;
  if (fabs(u - lo / P) < 1e-6 || fabs(u - hi / P) < 1e-6) out.fl |= DSDE_FLAG_SAMPLE_NEAR_TIE;
  return out;
}

__device__ __forceinline__ SeqRec load_seqrec(const SeqRec* p) {
  SeqRec r;
  r.mode = __ldcg(&p->mode);
  r.slot = __ldcg(&p->slot);
  r.trow = __ldcg(&p->trow);
  r.drow = __ldcg(&p->drow);
  r.M = __ldcg(&p->M);
  r.invT = __ldcg(&p->invT);
  r.C = __ldcg(&p->C);
  r.lam = __ldcg(&p->lam);
  r.u = __ldcg(&p->u);
  r.S = __ldcg(&p->S);
  return r;
}
