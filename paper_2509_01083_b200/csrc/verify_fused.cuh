// verify_fused.cuh — the whole verification step as ONE persistent kernel
// (included by verify.cu inside namespace dsde, after verify_draw.cuh).
//
// EXPERIMENTAL (DSDE_TAIL=fused; parity-green, NOT the default): measured
// ~360 us per cfg3 step against ~212 us for the stream kernel + k_tail, because
// the dependent latency chains of the tail work (row merge, finalize, draw,
// select) run inside a memory system saturated by the stream and slow the
// warps that carry them.
//
// k_fused: warps claim the a1 stream units (draft row r, slice u) in
// increasing order from a global counter, and the work that depends on them is
// done by whichever warp completes its inputs:
//   * the warp that writes the last slice partial of row r merges the row
//     (fp64), computes KL, log p/q and the Philox accept test (a2);
//   * the warp that merges the last row of sequence i finds a_i, writes the
//     KLDs and tokens, the draw record (a3), publishes a ready flag and, in the
//     whole-step launch, updates the signal and SL^ (a5-a6); the warp that
//     completes the last signal applies the batch cap and next SLs (a7);
//   * draw units (sequence i, slice u) are assigned statically to warps, in
//     sequence order; a warp takes its next one between stream units once the
//     sequence is ready; the warp completing the last unit of a sequence
//     selects the token (a4).
// Ordering: producers write with plain stores and bump a counter with a
// release atomic (atom.add.release.gpu: MEMBAR.ALL.GPU, no SC fence, no L1
// invalidation); the consumer that sees the final count issues an acquire
// fence and reads with ld.global.cg. Stream units are claimed dynamically, so
// a warp waiting for a ready flag never holds work that flag depends on (no
// co-residency requirement). A bad cu_sl cannot hang the kernel: the warp that
// merges the last row finalizes every sequence that did not complete as a
// data error, and a wait that never ends raises DSDE_DERR_STALL after ~2 s.

struct RowRes {  // 48 bytes, per draft row
  double kl, lam, C;
  float M;
  int flags;  // RR_* bits
  double pad0, pad1;
};
static_assert(sizeof(RowRes) == 48, "RowRes layout");
enum { RR_FINITE = 1, RR_ACCEPT = 2, RR_NEAR = 4, RR_BADTOK = 8 };

struct FusedCtl {  // zeroed before every launch; one 128-byte line per counter
  int rows_merged;
  int pad0[31];
  int q_tail;  // draw tasks published
  int pad1[31];
  int claim;  // draw units claimed
  int pad2[31];
  int sig_done;  // signals written (whole-step launch)
  int pad3[31];
};
// (q_tail / claim are unused since the static draw assignment; unit_next
// shares rows_merged's line padding slot 16 so the block stays 512 bytes)
#define FUSED_UNIT_NEXT(ctl) (&(ctl)->pad0[15])
static_assert(sizeof(FusedCtl) == kCtlInts * sizeof(int), "FusedCtl layout");

struct FusedArgs {
  int B, V, total, nsub, nd;
  const int32_t* cu_sl;
  const int32_t* tokens;
  const void* tl;
  long long ld_t;
  const void* dl;
  long long ld_d;
  const uint64_t* seeds;
  SubPartial* part;
  RowRes* rowres;
  SeqRec* rec;
  double* smass;
  float* sref;
  int32_t* acc_len;
  int32_t* emitted;
  float* kld;
  uint8_t* flags;
  int32_t* err;
  FusedCtl* ctl;
  int* row_cnt;   // [total]
  int* seq_cnt;   // [B]
  int* draw_cnt;  // [B]
  int* fin;       // [B]
  int* queue;     // [B] 1 once sequence i's draw record is published
  int step;       // 1: signal (+ cap if fuse_cap) fused
  int fuse_cap;
  SignalArgs sig;
  CapArgs cap;
};

__device__ __forceinline__ int ld_volatile(const int* p) { return *reinterpret_cast<const volatile int*>(p); }


// Release increment (MEMBAR.ALL.GPU + ATOM, no sequentially consistent fence
// and no L1 invalidation): the caller's prior writes are visible to whoever
// observes the new count.
__device__ __forceinline__ int atomic_add_release(int* p, int v) {
  int old;
  asm volatile("atom.add.release.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
// Acquire side after observing a final count (reads then use ld.global.cg).
__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// the sequence range of i, and whether it is well formed (as finalize_seq)
__device__ __forceinline__ bool seq_range(const FusedArgs& a, int i, int& c0, int& k) {
  c0 = __ldg(a.cu_sl + i);
  const int c1 = __ldg(a.cu_sl + i + 1);
  k = c1 - c0;
  const bool range_ok = c0 >= 0 && k >= 1 && k <= DSDE_MAX_SL && c1 <= a.total;
  const bool rows_ok = (i != a.B - 1) || (c1 == a.total);
  return range_ok && rows_ok;
}

// ---- a2: merge of row r's slice partials (lanes over slices), KL, accept test
template <typename T>
__device__ __noinline__ void merge_row(const FusedArgs& a, int r, int i) {
  const int lane = threadIdx.x & 31;
  const int nc = a.nsub;
  const SubPartial* P = a.part + (long long)r * nc;
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
    const float4 q0 = __ldcg(reinterpret_cast<const float4*>(P + c));
    const float4 q1 = __ldcg(reinterpret_cast<const float4*>(P + c) + 1);
    const double qS = q0.x, qA = q0.y, qD = q0.z, qM = q0.w, qC = q1.x;
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
  if (lane != 0) return;
  const double y = (D - A) / S;
  const double lam = log1p(y);
  const double kl = fmax(0.0, y <= 1.0 ? D / S + (lam - y) : A / S + lam);
  bool fin = isfinite(S) && isfinite(A) && isfinite(D) && S > 0.0 && isfinite(M) && isfinite(C) &&
             isfinite(kl);
  int flags = 0;
  int c0, k;
  if (seq_range(a, i, c0, k) && r >= c0 && r < c0 + k) {
    // accept test of position j = r - c0 (slot cu_sl[i] + i + j)
    const int x = __ldg(a.tokens + r);
    const bool bad_tok = x < 0 || x >= a.V;
    double lr = 0.0;
    if (!bad_tok) {
      const T* tp = reinterpret_cast<const T*>(a.tl) + ((long long)r + i) * a.ld_t;
      const T* dp = reinterpret_cast<const T*>(a.dl) + (long long)r * a.ld_d;
      const double tx = (double)load_logit<T>(tp + x), dx = (double)load_logit<T>(dp + x);
      lr = (tx - dx) - C + lam;
      fin = fin && isfinite(lr);
    }
    const Uniforms u = philox_uniforms(__ldg(a.seeds + (long long)r + i));
    const double pacc = lr >= 0.0 ? 1.0 : exp(lr);
    if (u.acc < pacc) flags |= RR_ACCEPT;
    if (fabs(u.acc - pacc) < 1e-6) flags |= RR_NEAR;
    if (bad_tok) flags |= RR_BADTOK;
  }
  if (fin) flags |= RR_FINITE;
  RowRes rr;
  rr.kl = kl;
  rr.lam = lam;
  rr.C = C;
  rr.M = Ml;
  rr.flags = flags;
  rr.pad0 = rr.pad1 = 0.0;
  a.rowres[r] = rr;
}

// ---- a5-a7 after sequence i's results are written; then publish its draw task
__device__ __noinline__ void seq_epilogue(const FusedArgs& a, int i) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
  // the draw record (and this warp's outputs) before the ready flag: the draw
  // of sequence i can start while its signal is computed
  if (lane == 0) atomic_add_release(a.queue + i, 1);
  if (a.step) {
    signal_seq(a.sig, i);
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomic_add_release(&a.ctl->sig_done, 1) == a.B - 1;
    last = __shfl_sync(kFull, last, 0);
    if (last && a.fuse_cap) {
      fence_acquire();
      cap_warp(a.cap);
    }
  }
}

// ---- a3: sequence i from its merged rows (one warp, lane j = position j)
template <typename T>
__device__ __noinline__ void finalize_seq_fused(const FusedArgs& a, int i) {
  const int lane = threadIdx.x & 31;
  int c0, k;
  seq_range(a, i, c0, k);
  const long long slot0 = (long long)c0 + i;
  RowRes rr;
  rr.flags = 0;
  if (lane < k) {
    const RowRes* p = a.rowres + c0 + lane;
    rr.kl = __ldcg(&p->kl);
    rr.lam = __ldcg(&p->lam);
    rr.C = __ldcg(&p->C);
    rr.M = __ldcg(&p->M);
    rr.flags = __ldcg(&p->flags);
  }
  const unsigned bt = __ballot_sync(kFull, lane < k && (rr.flags & RR_BADTOK));
  const unsigned nf = __ballot_sync(kFull, lane < k && !(rr.flags & RR_FINITE));
  const unsigned am = __ballot_sync(kFull, lane < k && (rr.flags & RR_ACCEPT));
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
      a.rec[i] = r;
    }
    seq_epilogue(a, i);
    return;
  }
  const int acc_run = __ffs(~am) - 1;  // first rejected lane (lanes >= k never accept)
  const int aa = acc_run < k ? acc_run : k;
  if (lane < k) a.kld[c0 + lane] = (float)rr.kl;
  if (lane <= k) {
    a.emitted[slot0 + lane] = lane < aa ? __ldg(a.tokens + c0 + lane) : DSDE_PAD;
    if (a.flags)
      a.flags[slot0 + lane] = ((rr.flags & RR_NEAR) && lane <= aa && lane < k) ? DSDE_FLAG_ACCEPT_NEAR_TIE : 0;
  }
  if (lane == 0) a.acc_len[i] = aa;
  if (lane == aa) {
    r.slot = (int)(slot0 + aa);
    r.trow = slot0 + aa;
    r.u = philox_uniforms(__ldg(a.seeds + slot0 + aa)).smp;
    if (aa < k) {
      r.mode = MODE_RESIDUAL;
      r.drow = (long long)c0 + aa;
      r.M = rr.M;
      r.C = rr.C;
      r.lam = rr.lam;
    } else {
      r.mode = MODE_BONUS;
      r.drow = -1;
      r.M = 0.f;
      r.C = 0.0;
      r.lam = 0.0;
    }
    a.rec[i] = r;
  }
  seq_epilogue(a, i);
}

// a malformed sequence (bad cu_sl range, or rows that never completed)
__device__ __noinline__ void finalize_seq_error(const FusedArgs& a, int i) {
  const int lane = threadIdx.x & 31;
  if (lane == 0) {
    int c0, k;
    const int c1 = __ldg(a.cu_sl + i + 1);
    c0 = __ldg(a.cu_sl + i);
    k = c1 - c0;
    const bool range_ok = c0 >= 0 && k >= 1 && k <= DSDE_MAX_SL && c1 <= a.total;
    a.acc_len[i] = -1;
    raise_device_error(a.err, range_ok ? DSDE_DERR_ROWS : DSDE_DERR_BAD_SL, i);
    SeqRec r;
    r.mode = MODE_ERROR;
    r.slot = 0;
    r.trow = 0;
    r.drow = -1;
    r.M = 0.f;
    r.C = r.lam = r.u = 0.0;
    r.pad0 = 0;
    r.S = 0.0;
    a.rec[i] = r;
  }
  seq_epilogue(a, i);
}

// every row has been merged: sequences that cannot complete are data errors
__device__ __noinline__ void cleanup_incomplete(const FusedArgs& a) {
  const int lane = threadIdx.x & 31;
  fence_acquire();
  for (int base = 0; base < a.B; base += 32) {
    const int i = base + lane;
    bool mine = false;
    if (i < a.B) {
      int c0, k;
      const bool ok = seq_range(a, i, c0, k);
      if (!ok || __ldcg(a.seq_cnt + i) != k) mine = atomicCAS(a.fin + i, 0, 1) == 0;
    }
    unsigned m = __ballot_sync(kFull, mine);
    while (m) {
      const int l = __ffs(m) - 1;
      m &= m - 1;
      finalize_seq_error(a, base + l);
    }
  }
}

// stream unit done -> row r complete? -> sequence complete?
// row r is complete: merge it; is sequence i complete? are all rows merged?
template <typename T>
__device__ __noinline__ void row_done(const FusedArgs& a, int r, int i) {
  const int lane = threadIdx.x & 31;
  fence_acquire();
  merge_row<T>(a, r, i);
  __syncwarp();
  int c0, k;
  const bool ok = seq_range(a, i, c0, k);
  int done = 0, all_rows = 0;
  if (lane == 0) {
    if (ok && r >= c0 && r < c0 + k && atomic_add_release(a.seq_cnt + i, 1) == k - 1)
      done = atomicCAS(a.fin + i, 0, 1) == 0;
    // the sequence count before the row count (cleanup reads both)
    all_rows = atomic_add_release(&a.ctl->rows_merged, 1) == a.total - 1;
  }
  done = __shfl_sync(kFull, done, 0);
  all_rows = __shfl_sync(kFull, all_rows, 0);
  if (done) {
    fence_acquire();
    finalize_seq_fused<T>(a, i);
  }
  if (all_rows) cleanup_incomplete(a);
}

template <typename T>
__device__ __forceinline__ void after_unit(const FusedArgs& a, int r, int i) {
  const int lane = threadIdx.x & 31;
  int last = 0;
#ifdef DSDE_FUSED_RELAXED
  if (lane == 0) last = atomicAdd(a.row_cnt + r, 1) == a.nsub - 1;
#else
  if (lane == 0) last = atomic_add_release(a.row_cnt + r, 1) == a.nsub - 1;
#endif
  if (!__shfl_sync(kFull, last, 0)) return;
  row_done<T>(a, r, i);
}

// ---- a4: one draw unit c = (task c / nd, slice c % nd)
template <typename T>
__device__ __noinline__ void draw_unit_fused(const FusedArgs& a, long long c, int i) {
  constexpr int NVD = Traits<T>::NVD;
  const int lane = threadIdx.x & 31;
  const int u = (int)(c % a.nd);
  SeqRec r;
  const SeqRec* rp = a.rec + i;
  r.mode = __ldcg(&rp->mode);
  const bool draw = r.mode == MODE_RESIDUAL || r.mode == MODE_BONUS;
  if (draw) {
    r.slot = __ldcg(&rp->slot);
    r.trow = __ldcg(&rp->trow);
    r.drow = __ldcg(&rp->drow);
    r.M = __ldcg(&rp->M);
    r.C = __ldcg(&rp->C);
    r.lam = __ldcg(&rp->lam);
    r.u = __ldcg(&rp->u);
    DrawArgs da{a.B, a.V, a.nd, a.tl, a.ld_t, a.dl, a.ld_d, a.rec, a.smass, a.sref};
    const long long q = (long long)i * a.nd + u;
    uint4 rt[NVD], rd[NVD];
    const DrawUnit d = draw_unit_load<T>(da, (int)u, r, rt, rd);
    draw_unit_finish<T>(da.smass + q, da.sref + q, d, rt, rd);
  }
  __syncwarp();
  int last = 0;
  if (lane == 0) last = atomic_add_release(a.draw_cnt + i, 1) == a.nd - 1;
  if (__shfl_sync(kFull, last, 0) && draw) {
    fence_acquire();
    SelArgs sa{a.B, a.V, a.nd, a.tl, a.ld_t, a.dl, a.ld_d, a.rec, a.smass, a.sref, a.emitted, a.flags, a.err};
    select_seq<T>(sa, i, r, SelSrcGlobal{sa.smass + (long long)i * sa.nsub, sa.sref + (long long)i * sa.nsub});
  }
}

#ifndef DSDE_FUSED_MINB
#define DSDE_FUSED_MINB 3
#endif
constexpr int kFusedThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kFusedThreads, DSDE_FUSED_MINB) k_fused(FusedArgs a) {
  constexpr int NV = Traits<T>::NV;
  const int lane = threadIdx.x & 31;
  const long long W = (long long)gridDim.x * (kFusedThreads / 32);
  const long long gw = (long long)blockIdx.x * (kFusedThreads / 32) + (threadIdx.x >> 5);
  const long long n_draw = (long long)a.B * a.nd;
  // Draw units d = (sequence d / nd, slice d % nd) are assigned statically,
  // d = gw + m W, so a warp's units come in sequence order and each warp polls
  // only the ready flag of the sequence of its next unit (no shared hot spot).
  long long dnext = gw;
  auto ready = [&](int i) -> bool {
    int v = 0;
    if (lane == 0) v = ld_volatile(a.queue + i);
    return __shfl_sync(kFull, v, 0) != 0;
  };

  // ---- stream units (a1), claimed dynamically in increasing order (a slow
  // warp takes fewer units, so no row waits on a straggler); after each unit,
  // the next draw unit if its sequence is ready
  const long long n_units = (long long)a.total * a.nsub;
  int* unit_next = FUSED_UNIT_NEXT(a.ctl);
  int qc = 0;
  if (lane == 0) qc = atomicAdd(unit_next, 1);
  long long q = __shfl_sync(kFull, qc, 0);
  int seq = 0;
  while (q < n_units) {
    int qn = 0;
    if (lane == 0) qn = atomicAdd(unit_next, 1);  // the next claim, in flight during this unit
    const int r = (int)((unsigned)q / (unsigned)a.nsub);
    const int u = (int)q - r * a.nsub;
    seq = seq_of_row(a.cu_sl, a.B, seq, r);
    uint4 rt[NV], rd[NV];
    load_slice<T>(reinterpret_cast<const T*>(a.tl) + (long long)(r + seq) * a.ld_t, a.V, u, rt);
    load_slice<T>(reinterpret_cast<const T*>(a.dl) + (long long)r * a.ld_d, a.V, u, rd);
    store_partial(a.part + q, slice_stats<T>(rt, rd));
    after_unit<T>(a, r, seq);
#ifndef DSDE_FUSED_NODRAW_A
    if (dnext < n_draw) {
      const int i = (int)(dnext / a.nd);
      if (ready(i)) {
        fence_acquire();
        draw_unit_fused<T>(a, dnext, i);
        dnext += W;
      }
    }
#endif
    q = __shfl_sync(kFull, qn, 0);
  }
  // ---- the remaining draw units (a4); bug guard: a sequence that is never
  // published (~2 s) raises DSDE_DERR_STALL instead of hanging the device
  int spin = 0;
  while (dnext < n_draw) {
    const int i = (int)(dnext / a.nd);
    if (!ready(i)) {
      if (++spin > (1 << 21)) {
        if (lane == 0) raise_device_error(a.err, DSDE_DERR_STALL, i);
        return;
      }
      __nanosleep(1000);
      continue;
    }
    fence_acquire();
    draw_unit_fused<T>(a, dnext, i);
    dnext += W;
  }
}
