// verify_fused.cuh — a1-a4 of dsde_verify in ONE persistent launch (included by
// verify.cu inside namespace dsde; uses its helpers).
//
// Work list (static, derived from cu_sl alone): per sequence i a block of
//   [k_i * nc "stream" items (draft row, vocab chunk)] followed by
//   [nc "draw" items of sequence i - lag] (the residual row a or bonus row k of
//    an earlier sequence), and a tail block with the draw items of the last
//    `lag` sequences. q = blockIdx.x + j * gridDim.x sweeps it in order.
// Roles per CTA (2 CTAs/SM, cooperative launch so all CTAs are co-resident):
//   * producer warp: decodes items (warp-cooperative cursor over cu_sl), waits
//     until the sequence of a draw item is finalised (acquire flag), and fills a
//     3-stage ring of 32 KB stages with 1-D TMA bulk copies;
//   * 8 consumer warps: stream items -> warp partial (S, A, D about M, C = M -
//     max d, see k_stream_ws); draw items -> warp draw mass (residual
//     rho = e (1 - e^{-z}), bonus e^{t - m_w});
//   * merger warp: stream items -> chunk partial (fp64); when the last chunk of
//     a sequence lands (atomic counter) it runs finalize (a2-a3: fp64 row merge,
//     KL, Philox accept test, a_i, layout) and publishes the draw record; draw
//     items -> sub-chunk masses; when the last lands it runs select (a4: the
//     inverse CDF over the sub-chunk masses, then inside the crossing sub-chunk,
//     re-read from L2).
// The draw row of sequence i is re-read `lag` sequences after it was streamed,
// while it is still L2-resident; the bonus row is read once from HBM.

enum { IT_STREAM = 0, IT_RESID = 1, IT_BONUS = 2, IT_NONE = 3 };

struct FusedArgs {
  int B, V, nchunks, total, lag, exp_flags;
  const int32_t* cu_sl;
  const int32_t* tokens;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const uint64_t* seeds;
  int32_t* acc_len;
  int32_t* emitted;
  float* kld;
  uint8_t* flags;
  ChunkPartial* part;  // [total * nc]
  SeqRec* rec;         // [B]
  double* smass;       // [B * nc * 8] draw mass per warp sub-chunk
  float* sref;         // [B * nc * 8] its reference (bonus)
  int* counters;       // [3 * B + 2]: stream chunks done, draw chunks done, record published,
                       //   event-queue tail, head
  int* evq;            // [2 * B] finisher events (seq << 1 | kind), -1 = not yet written
  int32_t* err;
};

constexpr int kFzThreads = 32 * (kCWarps + 2);  // + producer warp, merger/finisher warp

// push a finisher event (kind 0 = finalize, 1 = select) onto the global queue
__device__ __forceinline__ void push_event(const FusedArgs& a, int seq, int kind) {
  const int pos = atomicAdd(a.counters + 3 * a.B, 1);
  __threadfence();
  atomicExch(a.evq + pos, (seq << 1) | kind);
}

struct DrawSlot {  // 16 bytes
  double m;
  float ref;
  int pad;
};

struct StageDesc {  // 16 bytes, written by the producer before the stage's arrive
  int type;         // IT_*
  int seq;          // sequence of the item
  int c;            // vocab chunk
  int j;            // stream: draft position
};

template <typename T>
__host__ __device__ constexpr int fused_smem() {
  return kWsStages * 2 * stage_row_bytes<T>() +                 // stages
         kWsStages * 2 * kCWarps * (int)sizeof(WarpPartial) +   // stream slot sets
         kWsStages * 2 * kCWarps * (int)sizeof(DrawSlot) +      // draw slot sets
         kWsStages * (int)sizeof(StageDesc) +                   // stage descriptors
         6 * kWsStages * 8;                                     // mbarriers
}

// SeqRec read past L1 (written by another SM in this launch)
__device__ __forceinline__ SeqRec load_rec_cg(const SeqRec* p) {
  SeqRec r;
  const int4* src = reinterpret_cast<const int4*>(p);
  int4* dst = reinterpret_cast<int4*>(&r);
#pragma unroll
  for (int q = 0; q < (int)(sizeof(SeqRec) / 16); ++q) dst[q] = __ldcg(src + q);
  return r;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// First item index of block i (i in [0, B]): stream items of sequences < i plus
// the draw items placed in blocks < i (block j >= lag holds those of j - lag).
__device__ __forceinline__ long long block_start(const FusedArgs& a, int i) {
  const int cu = i < a.B ? __ldg(a.cu_sl + i) : a.total;
  return (long long)a.nchunks * ((long long)cu + max(0, i - a.lag));
}

struct ItemInfo {
  int type;   // IT_STREAM, or a draw item (IT_RESID / IT_BONUS / IT_NONE once resolved)
  int seq;    // sequence of the item
  int j;      // stream: draft position
  int c;      // vocab chunk
};

// Warp-cooperative decode with a forward cursor `blk` (items only move forward
// for a given warp): the block containing q is the last i with start(i) <= q.
__device__ __forceinline__ ItemInfo decode_item(const FusedArgs& a, long long q, int& blk) {
  const int lane = threadIdx.x & 31;
  while (true) {
    const int i = blk + 1 + lane;
    const bool le = i <= a.B && block_start(a, i) <= q;
    const unsigned m = __ballot_sync(kFull, le);
    blk += __popc(m);
    if (m != kFull) break;
  }
  ItemInfo it;
  const long long off = q - block_start(a, blk);
  if (blk < a.B) {
    const int c0 = __ldg(a.cu_sl + blk);
    const int k = __ldg(a.cu_sl + blk + 1) - c0;
    if (off < (long long)k * a.nchunks) {
      it.type = IT_STREAM;
      it.seq = blk;
      it.j = (int)(off / a.nchunks);
      it.c = (int)(off - (long long)it.j * a.nchunks);
      return it;
    }
    it.type = IT_RESID;  // draw item; resolved against the record
    it.seq = blk - a.lag;
    it.j = 0;
    it.c = (int)(off - (long long)k * a.nchunks);
    return it;
  }
  const int idx = (int)(off / a.nchunks);
  it.type = IT_RESID;
  it.seq = max(0, a.B - a.lag) + idx;
  it.j = 0;
  it.c = (int)(off - (long long)idx * a.nchunks);
  return it;
}

// ---------------------------------------------------------------------------
// finalize (a2-a3) of sequence i by one warp; all chunk partials of its rows
// are complete and visible.
// ---------------------------------------------------------------------------
template <typename T>
__device__ void finalize_seq(const FusedArgs& a, int i) {
  const int lane = threadIdx.x & 31;
  const int c0 = __ldg(a.cu_sl + i), k = __ldg(a.cu_sl + i + 1) - c0;
  const long long slot0 = (long long)c0 + i;
  const int nc = a.nchunks;
  // row statistics: lane j ends up holding row j's (KL, lam, C, M, finite)
  double kl_j = 0.0, lam_j = 0.0, C_j = 0.0;
  float M_j = 0.f;
  bool fin_j = true;
  for (int j = 0; j < k; ++j) {
    const ChunkPartial* P = a.part + ((long long)c0 + j) * nc;
    float Ml = -INFINITY, Dl = -INFINITY;
    for (int c = lane; c < nc; c += 32) {
      Ml = max_nan(Ml, __ldcg(&P[c].M));
      Dl = fmaxf(Dl, __ldcg(&P[c].maxd));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Ml = max_nan(Ml, __shfl_xor_sync(kFull, Ml, o));
      Dl = fmaxf(Dl, __shfl_xor_sync(kFull, Dl, o));
    }
    const double M = (double)Ml, C = (double)(Ml - Dl);  // C is an fp32 value
    double S = 0.0, A = 0.0, D = 0.0;
    for (int c = lane; c < nc; c += 32) {
      const double qS = __ldcg(&P[c].S), qA = __ldcg(&P[c].A), qD = __ldcg(&P[c].D);
      const double ls = (double)__ldcg(&P[c].M) - M;
      const double s = exp(ls);
      const double dl = (double)__ldcg(&P[c].C) - C;
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
    // y = E_p[exp(-w)] - 1; KL = D/S + (log1p(y) - y), or A/S + log1p(y) for y > 1
    const double y = (D - A) / S;
    const double lam = log1p(y);
    const double kl = fmax(0.0, y <= 1.0 ? D / S + (lam - y) : A / S + lam);
    const bool fin = isfinite(S) && isfinite(A) && isfinite(D) && S > 0.0 && isfinite(M) &&
                     isfinite(C) && isfinite(kl);
    if (lane == j) {
      kl_j = kl;
      lam_j = lam;
      C_j = C;
      M_j = Ml;
      fin_j = fin;
    }
  }
  // per position: accept test (lane j), first rejection, layout
  double lr = 0.0;
  bool acc = false, near = false, bad_tok = false, nonfin = false;
  Uniforms u = {0.0, 0.0};
  if (lane <= k) u = philox_uniforms(__ldg(a.seeds + slot0 + lane));
  if (lane < k) {
    const long long drow = (long long)c0 + lane;
    const int x = __ldg(a.tokens + drow);
    bad_tok = x < 0 || x >= a.V;
    nonfin = !fin_j;
    if (!bad_tok) {
      const T* tp = reinterpret_cast<const T*>(a.tl) + (drow + i) * a.ld_t;
      const T* dp = reinterpret_cast<const T*>(a.dl) + drow * a.ld_d;
      const double tx = (double)load_logit<T>(tp + x), dx = (double)load_logit<T>(dp + x);
      lr = (tx - dx) - C_j + lam_j;
      nonfin |= !isfinite(lr);
    }
    const double pacc = lr >= 0.0 ? 1.0 : exp(lr);
    acc = u.acc < pacc;
    near = fabs(u.acc - pacc) < 1e-6;
  }
  const unsigned bt = __ballot_sync(kFull, bad_tok);
  const unsigned nf = __ballot_sync(kFull, nonfin);
  const unsigned am = __ballot_sync(kFull, acc);
  SeqRec r;
  r.pad0 = 0;
  r.pad1 = 0.0;
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
      a.rec[i] = r;
    }
  } else {
    const int acc_run = __ffs(~am) - 1;  // first rejected lane (lanes >= k never accept)
    const int aa = acc_run < k ? acc_run : k;
    if (lane < k) a.kld[c0 + lane] = (float)kl_j;
    if (lane <= k) {
      a.emitted[slot0 + lane] = lane < aa ? __ldg(a.tokens + c0 + lane) : DSDE_PAD;
      if (a.flags) a.flags[slot0 + lane] = (near && lane <= aa && lane < k) ? DSDE_FLAG_ACCEPT_NEAR_TIE : 0;
    }
    if (lane == 0) a.acc_len[i] = aa;
    if (lane == aa) {
      r.slot = (int)(slot0 + aa);
      r.trow = slot0 + aa;
      r.u = u.smp;
      if (aa < k) {
        r.mode = MODE_RESIDUAL;
        r.drow = (long long)c0 + aa;
        r.M = M_j;
        r.C = C_j;
        r.lam = lam_j;
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
  __syncwarp();
  __threadfence();
  if (lane == 0) st_release(a.counters + 2 * a.B + i, 1);  // record published
}

// ---------------------------------------------------------------------------
// draw weights of one lane over a 1024-token (bf16) / 512-token (fp32)
// sub-chunk u, token u*SUB + (v*32 + lane)*VEC + e, from raw words; returns the
// reference (residual: M of the row; bonus: warp max of t).
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ float draw_weights_raw(const uint4 (&rt)[Traits<T>::NV],
                                                  const uint4 (&rd)[Traits<T>::NV], bool resid,
                                                  float M, float Cf, double lam,
                                                  float (&w)[Traits<T>::VEC * Traits<T>::NV]) {
  constexpr int E = Traits<T>::VEC * Traits<T>::NV;
  if (resid) {
    const float lhi = (float)lam, llo = (float)(lam - (double)lhi);
    const float ML2 = M * kLog2e;
#pragma unroll
    for (int h = 0; h < E; h += 2) {
      const float2 tt = pair_of<T>(rt, h), dd = pair_of<T>(rd, h);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float tv = q ? tt.y : tt.x, dv = q ? dd.y : dd.x;
        const float ev = fast_exp2(fmaf(tv, kLog2e, -ML2));  // 0 for padding
        const float z = (diff_ref<T>(tv, dv, Cf) + lhi) + llo;
        float pz = -2.812654656736413e-06f;  // h(-z): tools/fit_g.py (degree 7, |u| <= 1)
        pz = fmaf(pz, z, 2.5358644052175805e-05f);
        pz = fmaf(pz, z, -1.9836986029986292e-04f);
        pz = fmaf(pz, z, 1.3885394437238574e-03f);
        pz = fmaf(pz, z, -8.33334494382143e-03f);
        pz = fmaf(pz, z, 4.166673496365547e-02f);
        pz = fmaf(pz, z, -1.666666716337204e-01f);
        pz = fmaf(pz, z, 0.5f);
        const float one_m = z < 1.f ? z * fmaf(-z, pz, 1.f) : 1.f - fast_exp2(-z * kLog2e);
        w[h + q] = (z > 0.f && ev > 0.f) ? ev * one_m : 0.f;
      }
    }
    return M;
  }
  float m = -INFINITY;
#pragma unroll
  for (int h = 0; h < E; h += 2) {
    const float2 tt = pair_of<T>(rt, h);
    m = max_nan(m, max_nan(tt.x, tt.y));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max_nan(m, __shfl_xor_sync(kFull, m, o));
  const float mL2 = m * kLog2e;
#pragma unroll
  for (int h = 0; h < E; h += 2) {
    const float2 tt = pair_of<T>(rt, h);
    w[h] = m <= -1e30f ? 0.f : fast_exp2(fmaf(tt.x, kLog2e, -mL2));
    w[h + 1] = m <= -1e30f ? 0.f : fast_exp2(fmaf(tt.y, kLog2e, -mL2));
  }
  return m <= -1e30f ? -INFINITY : m;
}

// raw words of sub-chunk u of a row, from global memory (select pass)
template <typename T>
__device__ __forceinline__ void load_sub_raw(const T* row, int V, int u, uint4 (&r)[Traits<T>::NV]) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, SUB = 32 * VEC * NV;
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

// mass of a lane's draw weights in the select pass's order: per vector, warp sums
template <typename T>
__device__ __forceinline__ double draw_mass(const float (&w)[Traits<T>::VEC * Traits<T>::NV]) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV;
  double m = 0.0;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += w[v * VEC + e];
    m += wsum_d((double)ls);
  }
  return m;
}

// ---------------------------------------------------------------------------
// select (a4) of sequence i by one warp; all sub-chunk masses are complete.
// ---------------------------------------------------------------------------
template <typename T>
__device__ void select_seq(const FusedArgs& a, int i) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, E = VEC * NV, SUB = 32 * VEC * NV;
  const int lane = threadIdx.x & 31;
  const SeqRec r = load_rec_cg(a.rec + i);
  const bool resid = r.mode == MODE_RESIDUAL;
  const int nsub = a.nchunks * kCWarps;
  const double* wmass = a.smass + (long long)i * nsub;
  const float* wref = a.sref + (long long)i * nsub;
  float Mg = -INFINITY;
  if (!resid) {
    for (int s0 = lane; s0 < nsub; s0 += 32) Mg = max_nan(Mg, __ldcg(wref + s0));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mg = max_nan(Mg, __shfl_xor_sync(kFull, Mg, o));
  }
  auto scale_of = [&](int s0) -> double {
    if (resid) return 1.0;
    const float ms = __ldcg(wref + s0);
    return ms == -INFINITY ? 0.0 : exp((double)ms - (double)Mg);
  };
  double R = 0.0;
  for (int s0 = lane; s0 < nsub; s0 += 32) R += scale_of(s0) * __ldcg(wmass + s0);
  R = wsum_d(R);
  uint8_t fl = 0;
  const T* tp = reinterpret_cast<const T*>(a.tl) + r.trow * a.ld_t;
  if (!(R > 0.0) || !isfinite(R)) {
    if (lane == 0) {
      if (resid && isfinite(R)) {
        // D7 fallback: residual mass 0 -> draw from p of the same target row
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
  int us = -1, ulast = -1;
  double base = 0.0, base_last = 0.0, cum = 0.0;
  for (int g = 0; g < nsub; g += 32) {
    const int s0 = g + lane;
    const double ms = s0 < nsub ? scale_of(s0) * __ldcg(wmass + s0) : 0.0;
    const double incl = wscan_d(ms, lane);
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
  uint4 rt[NV], rd[NV];
  load_sub_raw<T>(tp, a.V, us, rt);
  if (resid) load_sub_raw<T>(reinterpret_cast<const T*>(a.dl) + r.drow * a.ld_d, a.V, us, rd);
  float w[E];
  draw_weights_raw<T>(rt, rd, resid, r.M, (float)r.C, r.lam, w);
  int tok = -1, last_pos = -1;
  double lo = 0.0, hi = 0.0, lp_lo = 0.0, lp_hi = 0.0, vbase = base;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    float ls = 0.f;
#pragma unroll
    for (int e = 0; e < VEC; ++e) ls += w[v * VEC + e];
    const double incl = wscan_d((double)ls, lane);
    const double pre = vbase + f * (incl - (double)ls);
    int cand = -1, lpos = -1;
    double clo = 0.0, chi = 0.0, llo = 0.0, lhi = 0.0;
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
      if (w[v * VEC + e] > 0.f) {
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
    const unsigned bp = __ballot_sync(kFull, lpos >= 0);
    if (bp) {
      const int lp = 31 - __clz(bp);
      last_pos = tok_base + lp * VEC + __shfl_sync(kFull, lpos, lp);
      lp_lo = __shfl_sync(kFull, llo, lp);
      lp_hi = __shfl_sync(kFull, lhi, lp);
    }
    vbase += f * __shfl_sync(kFull, incl, 31);
  }
  if (tok < 0) {
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


__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// Takes one published finisher event, if any, and processes it (warp-wide).
// Events are finalize (a2-a3) or select (a4) of a sequence; any idle merger of
// any CTA can take any event, so a CTA that completes a sequence is not stalled
// by that sequence's finalize. Returns false if no event was available.
template <typename T>
__device__ bool take_event(const FusedArgs& a) {
  const int lane = threadIdx.x & 31;
  int got = -1;
  if (lane == 0) {
    volatile const int* ctl = a.counters + 3 * a.B;
    const int h = ctl[1], t = ctl[0];
    if (h < t && atomicCAS(a.counters + 3 * a.B + 1, h, h + 1) == h) got = h;
  }
  got = __shfl_sync(kFull, got, 0);
  if (got < 0) return false;
  int ev = -1;
  if (lane == 0)
    while ((ev = *reinterpret_cast<volatile const int*>(a.evq + got)) < 0) __nanosleep(64);
  ev = __shfl_sync(kFull, ev, 0);
  __threadfence();
  const int seq = ev >> 1;
  if ((ev & 1) == 0) {
    finalize_seq<T>(a, seq);
  } else if (__ldcg(&a.rec[seq].mode) != MODE_ERROR) {
    select_seq<T>(a, seq);
  }
  return true;
}

// ---------------------------------------------------------------------------
// the persistent kernel
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kFzThreads, kWsCtas) k_verify_fused(FusedArgs a) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, E = VEC * NV, CH = chunk_elems<T>();
  constexpr int ROWB = stage_row_bytes<T>();
  constexpr int SL = CH / kCWarps;
  extern __shared__ __align__(128) uint8_t smem[];
  WarpPartial* slots = reinterpret_cast<WarpPartial*>(smem + kWsStages * 2 * ROWB);
  DrawSlot* dslots = reinterpret_cast<DrawSlot*>(slots + kWsStages * 2 * kCWarps);
  StageDesc* sdesc = reinterpret_cast<StageDesc*>(dslots + kWsStages * 2 * kCWarps);
  uint64_t* full = reinterpret_cast<uint64_t*>(sdesc + kWsStages);
  uint64_t* consumed = full + kWsStages;
  uint64_t* ready = consumed + kWsStages;   // [stage][2]
  uint64_t* freeb = ready + 2 * kWsStages;  // [stage][2]
  const int nc = a.nchunks;
  const long long n_items = (long long)nc * ((long long)a.total + a.B);
  const int G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // cu_sl sanity (the work list is derived from it): cu_sl[0] = 0, k_i in
  // [1, DSDE_MAX_SL], cu_sl[B] = total. A malformed cu_sl invalidates the batch.
  __shared__ int s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
    const int k = __ldg(a.cu_sl + i + 1) - __ldg(a.cu_sl + i);
    if (k < 1 || k > DSDE_MAX_SL) s_bad = 1;
  }
  if (threadIdx.x == 0 && (__ldg(a.cu_sl) != 0 || __ldg(a.cu_sl + a.B) != a.total)) s_bad = 2;
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
  if (s_bad) {
    if (blockIdx.x == 0) {
      for (int i = threadIdx.x; i < a.B; i += blockDim.x) a.acc_len[i] = -1;
      if (threadIdx.x == 0) raise_device_error(a.err, s_bad == 1 ? DSDE_DERR_BAD_SL : DSDE_DERR_ROWS, 0);
    }
    return;
  }

  if (warp == kCWarps) {
    // ---------------- producer ----------------
    int blk = 0, s = 0;
    uint32_t round = 0;
    for (long long q = blockIdx.x; q < n_items; q += G) {
      ItemInfo it = decode_item(a, q, blk);
      long long trow = 0, drow = 0;
      if (it.type == IT_STREAM) {
        drow = (long long)__ldg(a.cu_sl + it.seq) + it.j;
        trow = drow + it.seq;
      } else {
        // wait until the record is published: a relaxed volatile poll (an
        // ld.acquire.gpu would invalidate this SM's L1 on every probe), then
        // one fence for acquire ordering
        if (lane == 0)
          while (*reinterpret_cast<volatile const int*>(a.counters + 2 * a.B + it.seq) == 0)
            __nanosleep(128);
        __syncwarp();
        __threadfence();
        const int mode = __ldcg(&a.rec[it.seq].mode);
        it.type = mode == MODE_RESIDUAL ? IT_RESID : mode == MODE_BONUS ? IT_BONUS : IT_NONE;
        trow = __ldcg(&a.rec[it.seq].trow);
        drow = __ldcg(&a.rec[it.seq].drow);
      }
      if (round > 0) mbar_wait(&consumed[s], (round - 1) & 1u);

      if (lane == 0) {
        StageDesc dsc;
        dsc.type = it.type;
        dsc.seq = it.seq;
        dsc.c = it.c;
        dsc.j = it.j;
        sdesc[s] = dsc;
        const int c0 = it.c * CH;
        const int n_el = min(CH, a.V - c0);
        const uint32_t bytes = (uint32_t)(n_el * (int)sizeof(T)) & ~15u;
        uint8_t* dst = smem + s * 2 * ROWB;
        if (it.type == IT_NONE || bytes == 0) {
          mbar_arrive(&full[s]);
        } else {
          const bool two = it.type != IT_BONUS;
          mbar_arrive_expect_tx(&full[s], (two ? 2 : 1) * bytes);
          bulk_g2s(dst, reinterpret_cast<const T*>(a.tl) + trow * a.ld_t + c0, bytes, &full[s]);
          if (two) bulk_g2s(dst + ROWB, reinterpret_cast<const T*>(a.dl) + drow * a.ld_d + c0, bytes, &full[s]);
        }
      }
      if (++s == kWsStages) {
        s = 0;
        ++round;
      }
    }
    return;
  }

  if (warp == kCWarps + 1) {
    // ---------------- merger / finisher ----------------
#ifdef DSDE_DEBUG_TIMING
    const unsigned long long t_start = gtimer();
    unsigned long long t_stream_done = 0, t_ev = 0;
    int n_ev = 0;
    bool in_stream = true;
#endif
    int blk = 0, s = 0;
    uint32_t round = 0;
    for (long long q = blockIdx.x; q < n_items; q += G) {
      const ItemInfo it = decode_item(a, q, blk);
      const uint32_t b = round & 1u, u = round >> 1;
#ifdef DSDE_DEBUG_TIMING
      if (in_stream && it.type != IT_STREAM) { t_stream_done = gtimer(); in_stream = false; }
#endif
      while (!mbar_test(&ready[2 * s + b], u & 1u)) {
#ifdef DSDE_DEBUG_TIMING
        const unsigned long long te = gtimer();
        if (take_event<T>(a)) { t_ev += gtimer() - te; ++n_ev; } else __nanosleep(32);
#else
        if (!take_event<T>(a)) __nanosleep(32);
#endif
      }
      if (it.type == IT_STREAM) {
        const WarpPartial* wp = slots + (s * 2 + b) * kCWarps;
        float Mr = -INFINITY, Dx = -INFINITY;
#pragma unroll
        for (int w = 0; w < kCWarps; ++w) {
          Mr = max_nan(Mr, wp[w].M);
          Dx = fmaxf(Dx, wp[w].maxd);
        }
        const WarpPartial p = wp[lane < kCWarps ? lane : 0];
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[2 * s + b]);
        const float Cc = Mr - Dx;
        double S = 0.0, A = 0.0, D = 0.0;
        if (lane < kCWarps) {
          const double ls = (double)p.M - (double)Mr;
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
        int last = 0;
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
          const long long row = (long long)__ldg(a.cu_sl + it.seq) + it.j;
          a.part[row * nc + it.c] = cp;
          __threadfence();
          const int k = __ldg(a.cu_sl + it.seq + 1) - __ldg(a.cu_sl + it.seq);
          last = atomicAdd(a.counters + it.seq, 1) == k * nc - 1;
        }
        if (lane == 0 && last) push_event(a, it.seq, 0);
      } else {
        const DrawSlot* ds = dslots + (s * 2 + b) * kCWarps;
        const int ity = ds[0].pad;  // item type posted by the consumers
        const DrawSlot p = ds[lane < kCWarps ? lane : 0];
        __syncwarp();
        if (lane == 0) mbar_arrive(&freeb[2 * s + b]);
        if (ity != IT_NONE && lane < kCWarps) {
          const long long base = ((long long)it.seq * nc + it.c) * kCWarps;
          a.smass[base + lane] = p.m;
          a.sref[base + lane] = p.ref;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0 && atomicAdd(a.counters + a.B + it.seq, 1) == nc - 1) push_event(a, it.seq, 1);
      }
      if (++s == kWsStages) {
        s = 0;
        ++round;
      }
    }
    // all own items merged: help with the remaining finisher events
#ifdef DSDE_DEBUG_TIMING
    const unsigned long long t_items = gtimer();
#endif
    while (true) {
#ifdef DSDE_DEBUG_TIMING
      const unsigned long long te = gtimer();
      if (take_event<T>(a)) { t_ev += gtimer() - te; ++n_ev; continue; }
#else
      if (take_event<T>(a)) continue;
#endif
      if (*reinterpret_cast<volatile const int*>(a.counters + 3 * a.B + 1) >= 2 * a.B) break;
      __nanosleep(128);
    }
#ifdef DSDE_DEBUG_TIMING
    if (lane == 0)
      printf("T cta=%d start=%llu stream_done=%llu items_done=%llu end=%llu ev_ns=%llu n_ev=%d\n", blockIdx.x,
             t_start, t_stream_done, t_items, gtimer(), t_ev, n_ev);
#endif
    return;
  }

  // ---------------- consumers ----------------
  const float2 L2 = make_float2(kLog2e, kLog2e);
  const float2 K7 = make_float2(-2.812654656736413e-06f, -2.812654656736413e-06f);
  const float2 K6 = make_float2(2.5358644052175805e-05f, 2.5358644052175805e-05f);
  const float2 K5 = make_float2(-1.9836986029986292e-04f, -1.9836986029986292e-04f);
  const float2 K4 = make_float2(1.3885394437238574e-03f, 1.3885394437238574e-03f);
  const float2 K3 = make_float2(-8.33334494382143e-03f, -8.33334494382143e-03f);
  const float2 K2 = make_float2(4.166673496365547e-02f, 4.166673496365547e-02f);
  const float2 K1 = make_float2(-1.666666716337204e-01f, -1.666666716337204e-01f);
  const float2 K0 = make_float2(0.5f, 0.5f);
  int s = 0;
  uint32_t round = 0;
  for (long long q = blockIdx.x; q < n_items; q += G) {
    mbar_wait(&full[s], round & 1u);
    const StageDesc dsc = sdesc[s];

    const T* st = reinterpret_cast<const T*>(smem + s * 2 * ROWB);
    const T* sd = reinterpret_cast<const T*>(smem + s * 2 * ROWB + ROWB);
    const int c0 = dsc.c * CH;
    const int n_el = min(CH, a.V - c0);
    const bool two = dsc.type == IT_STREAM || dsc.type == IT_RESID;
    uint4 rt[NV], rd[NV];
    if (dsc.type != IT_NONE) {
      if (n_el == CH) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int e0 = warp * SL + (v * 32 + lane) * VEC;
          rt[v] = *reinterpret_cast<const uint4*>(st + e0);
          rd[v] = two ? *reinterpret_cast<const uint4*>(sd + e0) : rt[v];
        }
      } else {
        const int bulk_el = (int)(((uint32_t)(n_el * (int)sizeof(T)) & ~15u) / sizeof(T));
        long long trow = 0, drow = 0;
        if (bulk_el < n_el) {
          if (dsc.type == IT_STREAM) {
            drow = (long long)__ldg(a.cu_sl + dsc.seq) + dsc.j;
            trow = drow + dsc.seq;
          } else {
            trow = __ldcg(&a.rec[dsc.seq].trow);
            drow = __ldcg(&a.rec[dsc.seq].drow);
          }
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
              if (two) db[e] = sd[idx];
            } else if (idx < n_el) {
              tb[e] = reinterpret_cast<const T*>(a.tl)[trow * a.ld_t + c0 + idx];
              if (two) db[e] = reinterpret_cast<const T*>(a.dl)[drow * a.ld_d + c0 + idx];
            }
          }
          rt[v] = *reinterpret_cast<const uint4*>(tb);
          rd[v] = *reinterpret_cast<const uint4*>(db);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&consumed[s]);
    const uint32_t sb = round & 1u, su = round >> 1;

    if (dsc.type == IT_STREAM) {
      float mt = -INFINITY, md = -INFINITY;
      if constexpr (sizeof(T) == 2) {
        __nv_bfloat162 bt0 = *reinterpret_cast<const __nv_bfloat162*>(&rt[0].x), bt1 = bt0;
        __nv_bfloat162 bd0 = *reinterpret_cast<const __nv_bfloat162*>(&rd[0].x), bd1 = bd0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const uint32_t wt[4] = {rt[v].x, rt[v].y, rt[v].z, rt[v].w};
          const uint32_t wd[4] = {rd[v].x, rd[v].y, rd[v].z, rd[v].w};
#pragma unroll
          for (int h = 0; h < 4; h += 2) {
            bt0 = __hmax2_nan(bt0, *reinterpret_cast<const __nv_bfloat162*>(&wt[h]));
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
      float M, Dmax;
      if constexpr (sizeof(T) == 2) {
        __nv_bfloat162 pk = __floats2bfloat162_rn(mt, md);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const uint32_t y = __shfl_xor_sync(kFull, *reinterpret_cast<const uint32_t*>(&pk), o);
          pk = __hmax2_nan(pk, *reinterpret_cast<const __nv_bfloat162*>(&y));
        }
        M = __low2float(pk);
        const float dh = __high2float(pk);
        Dmax = dh == dh ? dh : warp_max(md);
      } else {
        M = warp_max(mt);
        Dmax = warp_max(md);
      }
      if (__any_sync(kFull, mt != mt)) M = NAN;
      WarpPartial p;
      if (M <= -1e30f) {
        p.S = p.A = p.D = 0.f;
        p.M = -INFINITY;
        p.C = 0.f;
        p.maxd = -INFINITY;
      } else {
        const float Cw = M - Dmax;
        const float ML2 = M * kLog2e, DL2 = Dmax * kLog2e;
        const float2 nML2 = make_float2(-ML2, -ML2), nDL2 = make_float2(-DL2, -DL2);
        float2 S2 = make_float2(0.f, 0.f), A2 = S2, D2 = S2;
#pragma unroll
        for (int h = 0; h < E; h += 2) {
          const float2 tt = pair_of<T>(rt, h), dd = pair_of<T>(rd, h);
          const float2 xt = __ffma2_rn(tt, L2, nML2);
          const float2 arg = __ffma2_rn(dd, L2, nDL2);
          const float2 e = make_float2(fast_exp2(xt.x), fast_exp2(xt.y));
          const float2 f = make_float2(fast_exp2(arg.x), fast_exp2(arg.y));
          const float2 w = diff2<T>(tt, dd, Cw);
          const float2 w2 = __fmul2_rn(w, w);
          float2 pp = __ffma2_rn(K7, w, K6);
          pp = __ffma2_rn(pp, w, K5);
          pp = __ffma2_rn(pp, w, K4);
          pp = __ffma2_rn(pp, w, K3);
          pp = __ffma2_rn(pp, w, K2);
          pp = __ffma2_rn(pp, w, K1);
          pp = __ffma2_rn(pp, w, K0);
          S2 = __fadd2_rn(S2, e);
          A2 = __ffma2_rn(e, w, A2);
          const float2 sm = __fmul2_rn(__fmul2_rn(e, w2), pp);
          const float2 bg = __ffma2_rn(e, w, __fadd2_rn(f, make_float2(-e.x, -e.y)));
          const float2 term =
              make_float2(fabsf(w.x) < 1.f ? sm.x : bg.x, fabsf(w.y) < 1.f ? sm.y : bg.y);
          D2 = __fadd2_rn(D2, term);
        }
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
    } else {
      DrawSlot p;
      p.m = 0.0;
      p.ref = -INFINITY;
      p.pad = dsc.type;
      if (dsc.type != IT_NONE) {
        const bool resid = dsc.type == IT_RESID;
        float Mr = 0.f, Cf = 0.f;
        double lam = 0.0;
        if (resid) {
          Mr = __ldcg(&a.rec[dsc.seq].M);
          Cf = (float)__ldcg(&a.rec[dsc.seq].C);
          lam = __ldcg(&a.rec[dsc.seq].lam);
        }
        float w[E];
        p.ref = draw_weights_raw<T>(rt, rd, resid, Mr, Cf, lam, w);
        p.m = draw_mass<T>(w);
      }
      if (lane == 0) {
        if (su > 0) mbar_wait(&freeb[2 * s + sb], (su - 1) & 1u);
        dslots[(s * 2 + sb) * kCWarps + warp] = p;
        mbar_arrive(&ready[2 * s + sb]);
      }
    }
    if (++s == kWsStages) {
      s = 0;
      ++round;
    }
  }
}
