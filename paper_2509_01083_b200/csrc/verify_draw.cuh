// verify_draw.cuh — a2-a4 of dsde_verify after the stream pass (included by
// verify.cu inside namespace dsde; uses its helpers).
//
//   k_finalize  one CTA per sequence, one warp per draft position: fp64 merge of
//               the row's chunk partials (lanes over chunks), KL, log p/q; then
//               warp 0 runs the Philox accept test of every position, finds the
//               first rejection a_i, lays out the emitted tokens and publishes
//               the draw record (residual row a_i, or the bonus row k_i) (a2-a3).
//   k_draw_ws   persistent CTAs with the same TMA ring as k_stream_ws over the
//               items (sequence, vocab chunk) of the draw rows: every consumer
//               warp forms the draw weights of its 1024-token (bf16) / 512-token
//               (fp32) sub-chunk and writes their mass (a4, first pass).
//   k_select    one warp per sequence: the inverse CDF over the sub-chunk
//               masses, then inside the crossing sub-chunk (re-read from L2)
//               in ascending token order (a4, D7).

enum { IT_RESID = 1, IT_BONUS = 2, IT_NONE = 3 };

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
  int32_t* err;
};

constexpr int kFinThreads = 32 * DSDE_MAX_SL;

template <typename T>
__global__ void __launch_bounds__(kFinThreads) k_finalize(FinArgs a) {
  __shared__ double s_kl[DSDE_MAX_SL], s_lam[DSDE_MAX_SL], s_C[DSDE_MAX_SL];
  __shared__ float s_M[DSDE_MAX_SL];
  __shared__ int s_fin[DSDE_MAX_SL];
  const int i = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c0 = __ldg(a.cu_sl + i), c1 = __ldg(a.cu_sl + i + 1);
  const int k = c1 - c0;
  const bool range_ok = c0 >= 0 && k >= 1 && k <= DSDE_MAX_SL && c1 <= a.total;
  const bool rows_ok = (i != a.B - 1) || (c1 == a.total);
  if (!range_ok || !rows_ok) {
    if (threadIdx.x == 0) {
      a.acc_len[i] = -1;
      a.rec[i].mode = MODE_ERROR;
      raise_device_error(a.err, range_ok ? DSDE_DERR_ROWS : DSDE_DERR_BAD_SL, i);
    }
    return;
  }
  const int nc = a.nchunks;
  if (warp < k) {
    // ---- row j = warp: fp64 merge about M = max_c M_c, C = fp32(M - max d) ----
    // Chunk c's w is shifted by Delta = C_c - C; with s = e^(M_c - M), E1 = s e^-Delta:
    //   S += s S_c,  A += s (A_c + S_c Delta),
    //   D += E1 D_c - A_c s expm1(-Delta) + S_c s g(Delta),  g(x) = expm1(-x) + x.
    const ChunkPartial* P = a.part + ((long long)c0 + warp) * nc;
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
    double S = 0.0, A = 0.0, D = 0.0;
    for (int c = lane; c < nc; c += 32) {
      const ChunkPartial q = P[c];
      const double ls = (double)q.M - M;
      const double s = exp(ls);
      const double dl = (double)q.C - C;
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
      S += s * q.S;
      A += s * q.A + s * q.S * dl;
      D += E1 * q.D - q.A * sem + q.S * sg;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      S += __shfl_xor_sync(kFull, S, o);
      A += __shfl_xor_sync(kFull, A, o);
      D += __shfl_xor_sync(kFull, D, o);
    }
    if (lane == 0) {
      // y = E_p[exp(-w)] - 1. KL = D/S + (log1p(y) - y) has no cancellation for
      // small KL; when y > 1 (the draft puts far more mass away from the
      // reference, e.g. disjoint supports) the equal form A/S + log1p(y) is used.
      const double y = (D - A) / S;
      const double lam = log1p(y);
      const double kl = fmax(0.0, y <= 1.0 ? D / S + (lam - y) : A / S + lam);
      s_kl[warp] = kl;
      s_lam[warp] = lam;
      s_C[warp] = C;
      s_M[warp] = Ml;
      s_fin[warp] = isfinite(S) && isfinite(A) && isfinite(D) && S > 0.0 && isfinite(M) &&
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
  if (lane <= k) u = philox_uniforms(__ldg(a.seeds + slot0 + lane));
  if (lane < k) {
    const long long drow = (long long)c0 + lane;
    const int x = __ldg(a.tokens + drow);
    bad_tok = x < 0 || x >= a.V;
    nonfin = !s_fin[lane];
    if (!bad_tok) {
      const T* tp = reinterpret_cast<const T*>(a.tl) + (drow + i) * a.ld_t;
      const T* dp = reinterpret_cast<const T*>(a.dl) + drow * a.ld_d;
      const double tx = (double)load_logit<T>(tp + x), dx = (double)load_logit<T>(dp + x);
      lr = (tx - dx) - s_C[lane] + s_lam[lane];
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
  if (lane == aa) {
    r.slot = (int)(slot0 + aa);
    r.trow = slot0 + aa;
    r.u = u.smp;
    if (aa < k) {
      r.mode = MODE_RESIDUAL;
      r.drow = (long long)c0 + aa;
      r.M = s_M[aa];
      r.C = s_C[aa];
      r.lam = s_lam[aa];
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
// k_select recomputes every weight bit-identically from the same words.
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

// mass of a lane's draw weights in the select pass's order: per vector, an
// fp32 lane sum, then an fp64 warp sum
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
// k_draw_ws: items q = (sequence i, vocab chunk c), q = i * nc + c, swept by
// persistent CTAs (q = blockIdx.x + j * grid). 1 TMA producer warp + 8
// consumer warps per CTA, a kWsStages ring of 2 x 16 KB (bf16) stages. The
// consumers write their sub-chunk mass and reference straight to global.
// ---------------------------------------------------------------------------
struct DrawArgs {
  int B, V, nchunks;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const SeqRec* rec;
  double* smass;  // [B * nc * 8]
  float* sref;    // [B * nc * 8]
};

constexpr int kDrawThreads = 32 * (kCWarps + 1);

template <typename T>
__host__ __device__ constexpr int draw_ws_smem() {
  return kWsStages * 2 * stage_row_bytes<T>() + kWsStages * 16 + 2 * kWsStages * 8;
}

template <typename T>
__global__ void __launch_bounds__(kDrawThreads, kWsCtas) k_draw_ws(DrawArgs a) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, E = VEC * NV, CH = chunk_elems<T>();
  constexpr int ROWB = stage_row_bytes<T>();
  constexpr int SL = CH / kCWarps;
  extern __shared__ __align__(128) uint8_t smem[];
  int4* sdesc = reinterpret_cast<int4*>(smem + kWsStages * 2 * ROWB);  // (type, seq, c, -)
  uint64_t* full = reinterpret_cast<uint64_t*>(sdesc + kWsStages);
  uint64_t* consumed = full + kWsStages;
  const int nc = a.nchunks;
  const long long n_items = (long long)a.B * nc;
  const int G = gridDim.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kWsStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&consumed[s], kCWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kCWarps) {
    // ---------------- TMA producer ----------------
    if (lane != 0) return;
    int s = 0;
    uint32_t round = 0;
    for (long long q = blockIdx.x; q < n_items; q += G) {
      const int i = (int)(q / nc), c = (int)(q - (long long)i * nc);
      const SeqRec* r = a.rec + i;
      const int mode = __ldg(&r->mode);
      const int type = mode == MODE_RESIDUAL ? IT_RESID : mode == MODE_BONUS ? IT_BONUS : IT_NONE;
      const long long trow = __ldg(&r->trow), drow = __ldg(&r->drow);
      if (round > 0) mbar_wait(&consumed[s], (round - 1) & 1u);
      sdesc[s] = make_int4(type, i, c, 0);
      const int c0 = c * CH;
      const int n_el = min(CH, a.V - c0);
      const uint32_t bytes = (uint32_t)(n_el * (int)sizeof(T)) & ~15u;
      uint8_t* dst = smem + s * 2 * ROWB;
      if (type == IT_NONE || bytes == 0) {
        mbar_arrive(&full[s]);
      } else {
        const bool two = type == IT_RESID;
        mbar_arrive_expect_tx(&full[s], (two ? 2 : 1) * bytes);
        bulk_g2s(dst, reinterpret_cast<const T*>(a.tl) + trow * a.ld_t + c0, bytes, &full[s]);
        if (two) bulk_g2s(dst + ROWB, reinterpret_cast<const T*>(a.dl) + drow * a.ld_d + c0, bytes, &full[s]);
      }
      if (++s == kWsStages) {
        s = 0;
        ++round;
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  int s = 0;
  uint32_t round = 0;
  for (long long q = blockIdx.x; q < n_items; q += G) {
    mbar_wait(&full[s], round & 1u);
    const int4 dsc = sdesc[s];
    const int type = dsc.x, i = dsc.y, c = dsc.z;
    const T* st = reinterpret_cast<const T*>(smem + s * 2 * ROWB);
    const T* sd = reinterpret_cast<const T*>(smem + s * 2 * ROWB + ROWB);
    const int c0 = c * CH;
    const int n_el = min(CH, a.V - c0);
    const bool resid = type == IT_RESID;
    uint4 rt[NV], rd[NV];
    if (type != IT_NONE) {
      if (n_el == CH) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int e0 = warp * SL + (v * 32 + lane) * VEC;
          rt[v] = *reinterpret_cast<const uint4*>(st + e0);
          rd[v] = resid ? *reinterpret_cast<const uint4*>(sd + e0) : rt[v];
        }
      } else {
        // last chunk: bulk-copied part, an unaligned tail from global, padding after V
        const int bulk_el = (int)(((uint32_t)(n_el * (int)sizeof(T)) & ~15u) / sizeof(T));
        const long long trow = __ldg(&a.rec[i].trow), drow = __ldg(&a.rec[i].drow);
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
              if (resid) db[e] = sd[idx];
            } else if (idx < n_el) {
              tb[e] = reinterpret_cast<const T*>(a.tl)[trow * a.ld_t + c0 + idx];
              if (resid) db[e] = reinterpret_cast<const T*>(a.dl)[drow * a.ld_d + c0 + idx];
            }
          }
          rt[v] = *reinterpret_cast<const uint4*>(tb);
          rd[v] = *reinterpret_cast<const uint4*>(db);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&consumed[s]);
    if (++s == kWsStages) {
      s = 0;
      ++round;
    }
    if (type == IT_NONE) continue;
    float Mr = 0.f, Cf = 0.f;
    double lam = 0.0;
    if (resid) {
      Mr = __ldg(&a.rec[i].M);
      Cf = (float)__ldg(&a.rec[i].C);
      lam = __ldg(&a.rec[i].lam);
    }
    float w[E];
    const float ref = draw_weights_raw<T>(rt, rd, resid, Mr, Cf, lam, w);
    const double m = draw_mass<T>(w);
    if (lane == 0) {
      const long long o = ((long long)i * nc + c) * kCWarps + warp;
      a.smass[o] = m;
      a.sref[o] = ref;
    }
  }
}

// ---------------------------------------------------------------------------
// k_select: one warp per sequence (4 per CTA).
// ---------------------------------------------------------------------------
struct SelArgs {
  int B, V, nchunks;
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

template <typename T>
__global__ void __launch_bounds__(128) k_select(SelArgs a) {
  constexpr int VEC = Traits<T>::VEC, NV = Traits<T>::NV, E = VEC * NV, SUB = 32 * VEC * NV;
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= a.B) return;
  const SeqRec r = a.rec[i];
  if (r.mode != MODE_RESIDUAL && r.mode != MODE_BONUS) return;
  const bool resid = r.mode == MODE_RESIDUAL;
  const int nsub = a.nchunks * kCWarps;
  const double* wmass = a.smass + (long long)i * nsub;
  const float* wref = a.sref + (long long)i * nsub;
  float Mg = -INFINITY;
  if (!resid) {
    for (int s0 = lane; s0 < nsub; s0 += 32) Mg = max_nan(Mg, wref[s0]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) Mg = max_nan(Mg, __shfl_xor_sync(kFull, Mg, o));
  }
  auto scale_of = [&](int s0) -> double {  // sub-chunk mass scale to the common reference
    if (resid) return 1.0;
    const float ms = wref[s0];
    return ms == -INFINITY ? 0.0 : exp((double)ms - (double)Mg);
  };
  double R = 0.0;
  for (int s0 = lane; s0 < nsub; s0 += 32) R += scale_of(s0) * wmass[s0];
  R = wsum_d(R);
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
  // crossing sub-chunk: first u with prefix(u) > target (fallback: last with mass)
  int us = -1, ulast = -1;
  double base = 0.0, base_last = 0.0, cum = 0.0;
  for (int g = 0; g < nsub; g += 32) {
    const int s0 = g + lane;
    const double ms = s0 < nsub ? scale_of(s0) * wmass[s0] : 0.0;
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
