// tail.cuh — k_tail: a2-a4 (and, in dsde_step, a5-a7) of the verification
// step after the row stream (included by verify.cu inside namespace dsde,
// after verify_draw.cuh).
//
// One CTA of NW warps per sequence i (grid-stride over the batch):
//   1. warp j < k_i merges draft row c0 + j's slice partials in fp64 and runs
//      its accept test (row_finalize, a2) -> RowRes in shared memory; with the
//      D23 recovery draw (p.proposal) a row that rejects its draft token also
//      gets its p CDF and its first proposal (spec_row);
//   2. warp 0 finds the first rejection a_i, writes the KLDs, the emitted-token
//      layout and the draw record of row a_i (residual) or k_i (bonus)
//      (seq_layout, a3);
//   3. D23 (p.proposal, recovery draws): the speculative first proposal or
//      rounds of proposals (tail_p_draw); otherwise (D7, or no proposal kept)
//      the warps sweep the vocabulary slices of the drawn row and record each
//      slice's draw-weight mass (draw_mass, a4 first pass); meanwhile, in
//      dsde_step, warp NW-1 first updates the sequence's signal and SL^
//      (signal_seq_vals, a5-a6) and the warp completing the batch's last
//      signal applies the cap (cap_warp, a7, single GPU);
//   4. warp 0 selects the token by the inverse CDF over the slice masses and
//      inside the crossing slice (select_seq, a4).
// The kernel is launched with programmatic dependent launch after the stream
// kernel: it becomes resident while the stream drains, checks the batch layout
// and waits (griddepcontrol.wait) before touching the stream's partials.

struct TailArgs {
  FinArgs fa;
  SelArgs sa;
  double* mass;  // [B * nsub] draw-weight mass per slice of the drawn row
  float* mref;   // [B * nsub] its reference
  int* ctl;      // [1] signals done (dsde_step, single GPU), zeroed by the stream kernel
  int step, fuse_cap;
  int no_draw;   // vocab-parallel finalize: stop after the layout, the draw record to fa.rec[i]
  SignalArgs sig;
  CapArgs cap;
  int proposal;  // D23 recovery draws (dsde_config.resample = DSDE_RESAMPLE_PROPOSAL, sampling)
};

__device__ __forceinline__ int atomic_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// a5-a7 of sequence i by one warp (dsde_step): the signal from the layout's
// values, then the batch cap by the warp whose signal completes the batch.
__device__ __forceinline__ void tail_signal(const TailArgs& p, int i, int k, double x, int acc, double h = 0.0) {
  if (!p.step) return;
  signal_seq_vals(p.sig, i, k, x, acc, h);
  __syncwarp();
  int last = 0;
  if ((threadIdx.x & 31) == 0) last = atomic_add_acq_rel(p.ctl, 1) == p.fa.B - 1;
  last = __shfl_sync(kFull, last, 0);
  if (last && p.fuse_cap) cap_warp(p.cap);
}

#ifndef DSDE_TAIL_TRACE
#define DSDE_TAIL_TRACE 0
#endif
#if DSDE_TAIL_TRACE
// measurement build only (-DDSDE_TAIL_TRACE=1): globaltimer stamps per CTA's
// first sequence: start, after the wait, finalize, layout, draw, select, smid
constexpr int kTraceMax = 8192;
__device__ unsigned long long g_tail_trace[kTraceMax * 8];
__device__ __forceinline__ void tail_stamp(int k) {
  if (threadIdx.x == 0 && blockIdx.x < kTraceMax) {
    unsigned long long t;
    // (the memory clobber keeps the read after a preceding __syncthreads: without
    // it ptxas may hoist the timer read above the barrier)
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    g_tail_trace[blockIdx.x * 8 + k] = t;
  }
}
#define TAIL_STAMP(k) tail_stamp(k)
#else
#define TAIL_STAMP(k) do {} while (0)
#endif

// D23's first proposal of a rejected draft row, by the row's finalize warp
// right after its finalize (speculative: the row is the recovery row only if
// no earlier row was rejected). Returns the kept token or -1; *fl gets its
// tie flags.
template <typename T>
__device__ __forceinline__ int first_proposal(const FinArgs& a, const PCdf& cdf, long long slot, long long drow_i,
                                              float invT, double C, double lam, uint8_t* fl) {
  const T* trow = reinterpret_cast<const T*>(a.tl) + slot * a.ld_t;
  const T* drow = reinterpret_cast<const T*>(a.dl) + drow_i * a.ld_d;
  const Uniforms U = philox_uniforms(__ldg(a.seeds + slot), 1u);  // (u_prop, u_keep) of proposal 1
  const PSel sel = p_select<T>(cdf, a.nsub, trow, a.V, invT, U.acc);
  int kept = 0;
  uint8_t f = sel.fl;
  if ((threadIdx.x & 31) == 0 && sel.tok >= 0) {
    const double z = ((double)sel.t - (double)load_logit<T>(drow + sel.tok)) * (double)invT - C + lam;
    const double keep = z > 0.0 ? -expm1(-z) : 0.0;  // max(0, p - q) / p at the proposal
    kept = U.smp < keep;
    if (fabs(U.smp - keep) < 1e-6) f |= DSDE_FLAG_SAMPLE_NEAR_TIE;
  }
  kept = __shfl_sync(kFull, kept, 0);
  *fl = (uint8_t)__shfl_sync(kFull, (int)f, 0);
  return kept ? sel.tok : -1;
}

// p's CDF of a sequence's draft rows on the D23 path, built during the
// finalize (k_tail phase 1) by the finalize warp of every row that rejects
// its draft token (at most kSpecSub stream slices), with the row's first
// proposal (speculative: it is the recovery row only if no earlier row
// rejected).
constexpr int kSpecSub = 64;
struct SpecRows {
  double pre[DSDE_MAX_SL][kSpecSub];
  float ml2[DSDE_MAX_SL][kSpecSub];
  double cdf[DSDE_MAX_SL][2];  // Mr, P
  int tok[DSDE_MAX_SL];        // the kept first proposal, or -1
  uint8_t fl[DSDE_MAX_SL];
};

// D23 speculation for draft row j of sequence i (one warp): the row's p CDF
// and its first proposal into the SpecRows entry j. (Out of line, the kernel
// parameters it references would need a per-thread local copy: 1.1 KB of
// stack.)
template <typename T>
__device__ __forceinline__ void spec_row(const FinArgs& a, int i, int c0, int j, double C, double lam, SpecRows* sp) {
  double Mr;
  const double P = pcdf_build(PRow{reinterpret_cast<const float*>(a.part + (long long)(c0 + j) * a.nsub), 8, 3},
                              a.nsub, sp->pre[j], sp->ml2[j], &Mr);
  __syncwarp();
  uint8_t f = 0;
  const int tk = first_proposal<T>(a, PCdf{sp->pre[j], sp->ml2[j], Mr, P}, (long long)c0 + i + j, (long long)c0 + j,
                                   inv_temp(a.temps, i), C, lam, &f);
  if ((threadIdx.x & 31) == 0) {
    sp->cdf[j][0] = Mr;
    sp->cdf[j][1] = P;
    sp->tok[j] = tk;
    sp->fl[j] = f;
  }
}

// a4 on the D23 path (p.proposal), a recovery draw (CTA-uniform result
// through *s_placed): p's CDF over the drawn row's stream slices (its draft
// row's partials) comes from the finalize's speculation (sp != NULL) or is
// built here by warp 0 into pre / ml2 (shared memory, or the workspace beyond
// kTailMaxSub slices); then proposals v_j ~ p (u_prop of proposal j), each
// kept iff u_keep < max(0, p_v - q_v) / p_v = -expm1(-z_v), z_v = log p_v/q_v
// = (t_v - d_v) / T - C + lam (the finalize's frame, in fp64): the speculative
// first proposal, then rounds of nwp proposals in parallel (one per warp; the
// signal warp of dsde_step is busy); the first kept j wins. *s_placed = 0 when
// the D7 draw must decide: no proposal kept in DSDE_RESAMPLE_PROPOSALS
// (flagged), or not a recovery draw (the bonus row is drawn by the D7 passes).
template <typename T, int NW>
__device__ void tail_p_draw(const TailArgs& p, int i, int aa, const SeqRec& r, const SpecRows* sp, double* pre,
                            float* ml2, double* s_cdf, int* s_ptok, uint8_t* s_pfl, int* s_placed) {
  const FinArgs& a = p.fa;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) *s_placed = 0;
  if (r.mode != MODE_RESIDUAL) return;
  const T* trow = reinterpret_cast<const T*>(a.tl) + r.trow * a.ld_t;
  uint8_t fl = sp ? sp->fl[aa] : 0;
  int tok = sp ? sp->tok[aa] : -1;  // the speculative first proposal
  if (tok >= 0) {
    if (threadIdx.x == 0) {
      a.emitted[r.slot] = tok;
      if (a.flags) a.flags[r.slot] |= fl;
      *s_placed = 1;
      if (i == (int)blockIdx.x) TAIL_STAMP(4);
    }
    return;
  }
  // the proposal warps synchronise among themselves (named barrier 1): the
  // signal warp of dsde_step runs concurrently and joins at the sequence's end
  const int nwp = NW - (p.step ? 1 : 0);
  if (warp >= nwp) return;  // the signal warp
  auto pbar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(nwp * 32) : "memory"); };
  if (!sp) {
    if (warp == 0) {
      double Mr;
      const double P = pcdf_build(PRow{reinterpret_cast<const float*>(a.part + r.drow * a.nsub), 8, 3}, a.nsub, pre,
                                  ml2, &Mr);
      if (lane == 0) {
        s_cdf[0] = Mr;
        s_cdf[1] = P;
      }
    }
    pbar();
  }
  const PCdf cdf = sp ? PCdf{const_cast<double*>(sp->pre[aa]), const_cast<float*>(sp->ml2[aa]), sp->cdf[aa][0],
                             sp->cdf[aa][1]}
                      : PCdf{pre, ml2, s_cdf[0], s_cdf[1]};
  const T* drow = reinterpret_cast<const T*>(a.dl) + r.drow * a.ld_d;
  const uint64_t seed = __ldg(a.seeds + r.slot);
  int j0_end = 0;
  for (int j0 = sp ? 2 : 1; j0 <= DSDE_RESAMPLE_PROPOSALS; j0 += nwp) {
    j0_end = j0;
    if (j0 + warp <= DSDE_RESAMPLE_PROPOSALS) {
      const Uniforms U = philox_uniforms(seed, (uint32_t)(j0 + warp));  // (u_prop, u_keep)
      const PSel sel = p_select<T>(cdf, a.nsub, trow, a.V, r.invT, U.acc);
      if (lane == 0) {
        int kept = 0;
        uint8_t f = sel.fl;
        if (sel.tok >= 0) {
          const double z = ((double)sel.t - (double)load_logit<T>(drow + sel.tok)) * (double)r.invT - r.C + r.lam;
          const double keep = z > 0.0 ? -expm1(-z) : 0.0;  // max(0, p - q) / p at the proposal
          kept = U.smp < keep;
          if (fabs(U.smp - keep) < 1e-6) f |= DSDE_FLAG_SAMPLE_NEAR_TIE;
        }
        s_ptok[warp] = kept ? sel.tok : -1;
        s_pfl[warp] = f;
      }
    }
    pbar();
    const int nr = min(nwp, DSDE_RESAMPLE_PROPOSALS + 1 - j0);
    for (int w = 0; w < nr; ++w) {  // the round's first kept proposal (same in every thread)
      fl |= s_pfl[w];
      if (s_ptok[w] >= 0) {
        tok = s_ptok[w];
        break;
      }
    }
    pbar();  // the records are rewritten by the next round
    if (tok >= 0) break;
  }
  (void)j0_end;
#if DSDE_TAIL_TRACE
  if (threadIdx.x == 0 && i == (int)blockIdx.x && blockIdx.x < kTraceMax) g_tail_trace[blockIdx.x * 8 + 7] = j0_end;
#endif
  if (threadIdx.x == 0) {
    if (tok >= 0) a.emitted[r.slot] = tok;
    if (a.flags) a.flags[r.slot] |= fl | (tok >= 0 ? 0 : DSDE_FLAG_PROPOSAL_FALLBACK);
    *s_placed = tok >= 0;
  }
  if (i == (int)blockIdx.x) TAIL_STAMP(4);
}

// draw slices per row whose records k_tail keeps in shared memory (V <= 262144
// bf16 / 131072 fp32; larger vocabularies use the workspace)
constexpr int kTailMaxSub = 256;

template <typename T, int NW>
__global__ void __launch_bounds__(NW * 32, 1024 / (NW * 32)) k_tail(TailArgs p) {
  const FinArgs& a = p.fa;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nd = p.sa.nsub;  // draw slices per row
  __shared__ RowRes s_rr[DSDE_MAX_SL];
  __shared__ SeqRec s_rec;
  __shared__ int s_acc, s_bad;
  __shared__ double s_mass[kTailMaxSub], s_scale[kTailMaxSub];
  __shared__ float s_ref[kTailMaxSub], s_wmax[NW];
  __shared__ int s_ptok[NW];
  __shared__ uint8_t s_pfl[NW];
  __shared__ double s_cdf[2];
  __shared__ int s_placed;
  // the D23 speculation records: dynamic shared memory, launched only with
  // p.proposal (a static 13 KB would change the D7 path's launch footprint)
  extern __shared__ __align__(16) unsigned char s_dyn[];
  SpecRows& s_sp = *reinterpret_cast<SpecRows*>(s_dyn);
  const bool smem = nd <= kTailMaxSub;
  // while the stream kernel drains: the batch check (cu_sl must be a
  // non-decreasing prefix from 0, else no row can be attributed to a sequence
  // and every sequence is a DSDE_DERR_BAD_SL error) and the accept-test
  // inputs of this CTA's first sequence (warp j: row j)
  if (warp == 0) {
    int bad = __ldg(a.cu_sl) != 0;
    for (int i = lane; i < a.B; i += 32) bad |= __ldg(a.cu_sl + i + 1) < __ldg(a.cu_sl + i);
    bad = __any_sync(kFull, bad);
    if (lane == 0) s_bad = bad;
  }
  TAIL_STAMP(0);
  RowPre pre{0, 0.f, 0.f, 0.0};
  int pre_i = -1;
  __shared__ double s_ubonus;  // u_smp of the first sequence's bonus slot
  {
    const int i = blockIdx.x, c0 = __ldg(a.cu_sl + i), k = __ldg(a.cu_sl + i + 1) - c0;
    if (k >= 1 && k <= DSDE_MAX_SL && c0 >= 0 && c0 + k <= a.total) {
      pre_i = i;
      if (warp < k) pre = row_prefetch<T>(a, c0 + warp, i);
      if (warp == min(k, NW - 1) && lane == 0 && !seq_greedy(a, i))
        s_ubonus = philox_uniforms(__ldg(a.seeds + (long long)c0 + i + k)).smp;
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  TAIL_STAMP(1);
  const bool all_bad = s_bad != 0;
  for (int i = blockIdx.x; i < a.B; i += gridDim.x) {
    int c0 = 0, k = 0;
    bool rows_ok = true;
    const bool ok = !all_bad && seq_ok(a, i, c0, k, &rows_ok);
    if (!ok) {
      // malformed sequence: accepted_len -1 and the device error; with
      // dsde_step it counts towards the cap (SL^ = sl_min, state untouched),
      // exactly as dsde_update_signal treats it
      if (warp == 0) {
        if (lane == 0) {
          a.acc_len[i] = -1;
          raise_device_error(a.err, rows_ok ? DSDE_DERR_BAD_SL : DSDE_DERR_ROWS, i);
          if (p.no_draw) a.rec[i] = error_rec(0);
        }
        tail_signal(p, i, 0, 0.0, -1);
      }
      continue;  // CTA-uniform
    }
    // 1. a2: row finalize, warp j -> draft row c0 + j
    // D23 speculation (p.proposal): the finalize warp of a row that rejects its
    // draft token also builds the row's p CDF and evaluates its first
    // proposal, so that the layout mostly finds the recovery token ready.
    const bool spec = p.proposal && a.nsub <= kSpecSub && !seq_greedy(a, i);
    for (int j = warp; j < k; j += NW) {
      const RowRes rr = row_finalize<T>(a, c0 + j, i, (i == pre_i && j == warp) ? &pre : nullptr);
      if (lane == 0) s_rr[j] = rr;
      // (only a row that rejects its draft token can be the recovery row)
      if (spec && (rr.bits & RR_FINITE) && !(rr.bits & (RR_ACCEPT | RR_BADTOK)))
        spec_row<T>(a, i, c0, j, rr.C, rr.lam, &s_sp);
    }
    __syncthreads();
    if (i == (int)blockIdx.x) TAIL_STAMP(2);
    // 2. a3: layout and draw record (warp 0)
    if (warp == 0) {
      RowRes rr;
      rr.bits = 0;
      rr.x = 0;
      rr.kl = 0.0;
      if (lane < k) rr = s_rr[lane];
      const int acc = seq_layout(a, i, c0, k, rr, &s_rec, i == pre_i ? &s_ubonus : nullptr);
      if (lane == 0) s_acc = acc;
    }
    __syncthreads();
    if (i == (int)blockIdx.x) TAIL_STAMP(3);
    const SeqRec r = s_rec;
    if (p.no_draw) {  // vocab-parallel: the shards draw from the published record
      if (threadIdx.x == 0) a.rec[i] = r;
      __syncthreads();
      continue;
    }
    // 3. a5-a7 (dsde_step) by the last warp, then a4's slice masses by all
    if (warp == NW - 1 && p.step) {
      const double x = lane < k ? (double)(float)s_rr[lane].kl : 0.0;  // the fp32 KLDs, as the 3-call path
      // the draft entropies the finalize warps wrote (D22), as the 3-call path reads them
      const double h = (p.sig.ent && lane < k && s_acc >= 0) ? (double)__ldcg(p.sig.ent + c0 + lane) : 0.0;
      tail_signal(p, i, k, x, s_acc, h);
    }
    // D23: the recovery token by proposals from p (CTA-uniform);
    // false: the D7 draw below (no proposal kept, or the D7 / greedy modes)
    // (p's CDF in the draw records' space: shared memory, or the workspace
    // beyond kTailMaxSub stream slices)
    bool placed = false;
    if (p.proposal) {
      tail_p_draw<T, NW>(p, i, s_acc, r, spec ? &s_sp : nullptr, a.nsub <= kTailMaxSub ? s_mass : p.mass + (long long)i * nd,
                         a.nsub <= kTailMaxSub ? s_ref : p.mref + (long long)i * nd, s_cdf, s_ptok, s_pfl, &s_placed);
      __syncthreads();
      placed = s_placed != 0;
    }
    if (!placed && (r.mode == MODE_RESIDUAL || r.mode == MODE_BONUS || r.mode == MODE_ARGMAX)) {
      const long long q0 = (long long)i * nd;
      double* gm = p.mass + q0;
      float* gr = p.mref + q0;
      if (r.mode == MODE_RESIDUAL) {
        for (int u = warp; u < nd; u += NW)
          draw_mass<T>(r, u, a.V, a.tl, a.ld_t, a.dl, a.ld_d, smem ? s_mass + u : gm + u, smem ? s_ref + u : gr + u);
      } else {  // t-only rows: slices u and u + NW per iteration
        for (int u = warp; u < nd; u += 2 * NW) {
          const int u1 = u + NW;
          draw_mass_t2<T>(r, u, u1, nd, a.V, a.tl, a.ld_t, smem ? s_mass + u : gm + u, smem ? s_ref + u : gr + u,
                          smem ? s_mass + u1 : gm + u1, smem ? s_ref + u1 : gr + u1);
        }
      }
      __syncthreads();
      if (i == (int)blockIdx.x) TAIL_STAMP(4);
      // 4. a4 select (warp 0)
      if (!smem) {
        if (warp == 0) select_seq<T, false>(p.sa, i, r, SliceSrc<false>{gm, gr, nullptr});
      } else {
        if (r.mode == MODE_BONUS) {
          // the whole CTA rescales the bonus slice masses to the row max Mg (one
          // fp64 exp per slice, in parallel), as select_seq would slice by slice
          // (s_ref holds the raw slice maxima m; the references are fl32(m / T))
          float mg = -INFINITY;
          for (int u = threadIdx.x; u < nd; u += NW * 32) mg = max_nan(mg, s_ref[u]);
          mg = warp_max_nan(mg);
          if (lane == 0) s_wmax[warp] = mg;
          __syncthreads();
          float Mg = s_wmax[0];
#pragma unroll
          for (int w = 1; w < NW; ++w) Mg = max_nan(Mg, s_wmax[w]);
          Mg = __fmul_rn(Mg, r.invT);
          for (int u = threadIdx.x; u < nd; u += NW * 32) {
            const float ms = s_ref[u];
            const double f = ms == -INFINITY ? 0.0 : exp((double)__fmul_rn(ms, r.invT) - (double)Mg);
            s_scale[u] = f;
            s_mass[u] = f * s_mass[u];
          }
          __syncthreads();
        }
        if (warp == 0) select_seq<T, true>(p.sa, i, r, SliceSrc<true>{s_mass, s_ref, s_scale});
#if DSDE_TAIL_TRACE == 2
        // measurement only: the select again (warm instructions and data), its
        // duration in slot 7
        if (warp == 0 && i == (int)blockIdx.x && blockIdx.x < kTraceMax) {
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
          select_seq<T, true>(p.sa, i, r, SliceSrc<true>{s_mass, s_ref, s_scale});
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
          if (lane == 0) g_tail_trace[blockIdx.x * 8 + 7] = t1 - t0;
        }
#endif
#if DSDE_TAIL_TRACE == 3
        // measurement only: the draw pass again over the previous sequence's
        // bonus row (warm instructions, cold data), its duration in slot 7
        if (r.mode == MODE_BONUS && i == (int)blockIdx.x && i > 0 && blockIdx.x < kTraceMax) {
          __syncthreads();
          unsigned long long t0, t1;
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
          SeqRec r2 = r;
          r2.trow = (long long)__ldg(a.cu_sl + i) + i - 1;  // the bonus row of sequence i - 1
          for (int u = warp; u < nd; u += 2 * NW)
            draw_mass_t2<T>(r2, u, u + NW, nd, a.V, a.tl, a.ld_t, s_mass + u, s_ref + u, s_mass + u + NW, s_ref + u + NW);
          __syncthreads();
          asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
          if (threadIdx.x == 0) g_tail_trace[blockIdx.x * 8 + 7] = t1 - t0;
        }
#endif
      }
    }
    __syncthreads();  // shared records are reused by the next sequence
    if (i == (int)blockIdx.x) {
      TAIL_STAMP(5);
#if DSDE_TAIL_TRACE
      if (threadIdx.x == 0 && blockIdx.x < kTraceMax) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_tail_trace[blockIdx.x * 8 + 6] = ((unsigned long long)smid << 8) | (unsigned)r.mode;
      }
#endif
    }
  }
}
