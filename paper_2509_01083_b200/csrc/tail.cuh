// tail.cuh — k_tail: a2-a4 (and, in dsde_step, a5-a7) of the verification
// step after the row stream (included by verify.cu inside namespace dsde,
// after verify_draw.cuh).
//
// One CTA of NW warps per sequence i (grid-stride over the batch):
//   1. warp j < k_i merges draft row c0 + j's slice partials in fp64 and runs
//      its accept test (row_finalize, a2) -> RowRes in shared memory;
//   2. warp 0 finds the first rejection a_i, writes the KLDs, the emitted-token
//      layout and the draw record of row a_i (residual) or k_i (bonus)
//      (seq_layout, a3);
//   3. the warps sweep the vocabulary slices of the drawn row and record each
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
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_tail_trace[blockIdx.x * 8 + k] = t;
  }
}
#define TAIL_STAMP(k) tail_stamp(k)
#else
#define TAIL_STAMP(k) do {} while (0)
#endif

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
    for (int j = warp; j < k; j += NW) {
      const RowRes rr = row_finalize<T>(a, c0 + j, i, (i == pre_i && j == warp) ? &pre : nullptr);
      if (lane == 0) s_rr[j] = rr;
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
    if (r.mode == MODE_RESIDUAL || r.mode == MODE_BONUS || r.mode == MODE_ARGMAX) {
      const long long q0 = (long long)i * nd;
      double* gm = p.mass + q0;
      float* gr = p.mref + q0;
      for (int u = warp; u < nd; u += NW)
        draw_mass<T>(r, u, a.V, a.tl, a.ld_t, a.dl, a.ld_d, smem ? s_mass + u : gm + u, smem ? s_ref + u : gr + u);
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
