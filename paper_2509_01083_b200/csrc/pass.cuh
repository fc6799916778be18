// pass.cuh — the whole verification step (a1-a4, with dsde_step also a5-a7)
// as ONE persistent kernel, k_pass (included by verify.cu inside namespace
// dsde, after verify_draw.cuh). The default path of dsde_verify / dsde_step.
//
// Why one kernel: after the row stream (a1, HBM-bound) every sequence needs a
// short chain of dependent, latency-bound work — merge its rows (a2), find the
// first rejection (a3), draw its token from the residual or bonus row (a4) —
// and the drawn row must be read again. Run after the stream, that chain is a
// serial tail of the step (round 1: 28% of config 3); interleaved with the
// stream of later sequences it is hidden, and the drawn rows, streamed a few
// microseconds earlier, are re-read from L2 instead of HBM.
//
// Work of warp gw (of W), iteration j, "unit" q = gw + j W (row r = q / nsub,
// vocabulary slice u = q % nsub), for q < (n_rows + Ld) nsub:
//   1. deferred tasks (below) whose inputs are complete by now;
//   2. attached row finalize: if u == (r - Lr) % nsub, row r - Lr is merged in
//      fp64 and its accept test run (a2) once all its slices are in; the warp
//      finalizing a sequence's last row lays the sequence out (a3), publishes
//      its draw record and, in dsde_step, updates its signal and SL^ (a5-a6);
//      the warp completing the batch's last signal applies the cap (a7);
//   3. attached draw: if row r - Ld is the LAST row of a sequence i, the
//      draw-weight mass of slice u of i's drawn row (a4, first pass) once the
//      record is published; the warp completing the last of the nsub slices
//      selects the token (a4);
//   4. stream unit (r < n_rows): the slice statistics of the row pair (a1),
//      then a release increment of the row's slice count.
// The finalize and draw work is thus spread deterministically over all warps
// instead of falling to whichever warp completes a row (that warp, delayed by
// the finalize, would tend to complete the next row too: a convoy). A task
// whose inputs are not complete is deferred to a per-warp FIFO and run as soon
// as they are, so the stream never stalls on the finalize chain; a warp waits
// only when its FIFO is full or after its last stream unit, and then only on
// work of strictly earlier iterations (Lr = ceil(W / nsub) + 1 rows puts a
// row's slices at least one iteration before its finalize, Ld = 2 Lr + 1 the
// sequence's finalizes before its draws), so with every warp resident (the
// grid is the occupancy-derived resident size) the kernel cannot deadlock; a
// bug guard raises DSDE_DERR_STALL after ~2 s.
// Counters (zeroed per call by the host): row_cnt[row], seq_cnt[i],
// draw_cnt[i], pub[i], ctl[0] = signals done.

struct PassArgs {
  FinArgs fa;        // rows, sequences, outputs (verify_draw.cuh)
  SelArgs sa;
  RowRes* rowres;    // [total]
  double* mass;      // [B * nsub] draw-weight mass per slice of the drawn row
  float* mref;       // [B * nsub] its reference
  int* row_cnt;      // [total]
  int* seq_cnt;      // [B]
  int* draw_cnt;     // [B]
  int* pub;          // [B]  1 once sequence i's draw record is published
  int* ctl;          // [8]  ctl[0]: signals done (dsde_step)
  int Lr, Ld;        // row-finalize and draw lags in rows
  int step, fuse_cap;
  SignalArgs sig;
  CapArgs cap;
};

#ifndef DSDE_PASS_TRACE
#define DSDE_PASS_TRACE 0
#endif
#if DSDE_PASS_TRACE
// measurement build only (-DDSDE_PASS_TRACE=1): per-warp and per-sequence
// globaltimer stamps / counts, read back by dsde_debug_pass_trace
constexpr int kTraceWarps = 8192, kTraceSeqs = 4096;
__device__ unsigned long long g_warp_trace[kTraceWarps * 8];  // start, loop end, end, wait ns, defers, rowfin, seqfin, draws
__device__ unsigned long long g_seq_trace[kTraceSeqs * 4];    // last row done, published, selected, -
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ long long trace_gw() {
  return (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
}
#define WTRACE_SET(k, v) \
  do { if ((threadIdx.x & 31) == 0 && trace_gw() < kTraceWarps) g_warp_trace[trace_gw() * 8 + (k)] = (v); } while (0)
#define WTRACE_ADD(k, v) \
  do { if ((threadIdx.x & 31) == 0 && trace_gw() < kTraceWarps) g_warp_trace[trace_gw() * 8 + (k)] += (v); } while (0)
#define STRACE_SET(i, k) \
  do { if ((threadIdx.x & 31) == 0 && (i) < kTraceSeqs) g_seq_trace[(i) * 4 + (k)] = gtimer(); } while (0)
#else
#define WTRACE_SET(k, v) do {} while (0)
#define WTRACE_ADD(k, v) do {} while (0)
#define STRACE_SET(i, k) do {} while (0)
#endif

__device__ __forceinline__ int atomic_add_release(int* p, int v) {
  int old;
  asm volatile("atom.add.release.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Lane 0 adds 1 to *cnt with release semantics (the warp's prior writes are
// made visible at L2 before the count); true in every lane if this was the
// n-th arrival. Memory ordering on the reading side: everything this kernel
// writes for another warp is read with ld.global.cg / ld.relaxed.gpu (L2, the
// point of coherence), issued only after the count (or flag) that orders it
// was observed — no acquire fence, because a gpu-scope acquire invalidates the
// whole L1 of the SM (CCTL.IVALL) and the stream's spilled loop state with it.
__device__ __forceinline__ bool arrive_last(int* cnt, int n) {
  __syncwarp();
  int last = 0;
  if ((threadIdx.x & 31) == 0) last = atomic_add_release(cnt, 1) == n - 1;
  last = __shfl_sync(kFull, last, 0);
  __syncwarp();
  return last != 0;
}

// a5-a7 of sequence i (dsde_step): the signal from the layout's values, then
// the batch cap by the warp completing the last signal (single GPU).
__device__ __noinline__ void pass_signal(const PassArgs& p, int i, int k, double x, int acc) {
  if (!p.step) return;
  signal_seq_vals(p.sig, i, k, x, acc);
  if (arrive_last(p.ctl + 0, p.fa.B) && p.fuse_cap) cap_warp(p.cap);
}

// a3 by the warp that completed sequence i's last row; then publish the draw.
__device__ __noinline__ void pass_seq(const PassArgs& p, int i, int c0, int k) {
  const int lane = threadIdx.x & 31;
  RowRes rr;
  rr.bits = 0;
  rr.kl = 0.0;
  if (lane < k) rr = load_rowres(p.rowres + c0 + lane);
  STRACE_SET(i, 0);
  WTRACE_ADD(6, 1);
  const int acc = seq_layout(p.fa, i, c0, k, rr, p.fa.rec + i);
  __syncwarp();
  if (lane == 0) st_release(p.pub + i, 1);
  STRACE_SET(i, 1);
  // the signal reads the KLDs as the three-call path does: the fp32 values
  pass_signal(p, i, k, (double)(float)rr.kl, acc);
}

// a2 of row r of sequence i (by the warp the row's finalize is attached to,
// once all its slices are in); the warp finalizing the sequence's last row
// lays the sequence out.
template <typename T>
__device__ __noinline__ void pass_row(const PassArgs& p, int r, int i) {
  int c0, k;
  if (!seq_ok(p.fa, i, c0, k) || r < c0 || r >= c0 + k) return;  // reported by pass_invalid
  WTRACE_ADD(5, 1);
  const RowRes rr = row_finalize<T>(p.fa, r, i);
  store_rowres(p.rowres + r, rr);
  if (arrive_last(p.seq_cnt + i, k)) pass_seq(p, i, c0, k);
}

// a4: slice u of sequence i's drawn row (published); the warp completing the
// last slice selects the token.
template <typename T>
__device__ __noinline__ void pass_draw(const PassArgs& p, int i, int u) {
  WTRACE_ADD(7, 1);
  const SeqRec r = load_seqrec(p.fa.rec + i);
  const long long q = (long long)i * p.fa.nsub + u;
#if DSDE_PASS_EXP != 4
  draw_mass<T>(r, u, p.fa.V, p.fa.tl, p.fa.ld_t, p.fa.dl, p.fa.ld_d, p.mass + q, p.mref + q);
#endif
  if (arrive_last(p.draw_cnt + i, p.fa.nsub)) {
    select_seq<T>(p.sa, i, r, p.mass + (long long)i * p.fa.nsub, p.mref + (long long)i * p.fa.nsub);
    STRACE_SET(i, 2);
  }
}

// Attached tasks (a row finalize, a draw unit) whose inputs are not complete
// when the warp reaches them wait in small per-warp FIFOs in shared memory,
// one per kind (rows complete, and sequences are published, nearly in order,
// so a FIFO head is the next to become ready and no kind blocks the other),
// and are run as soon as they are: a warp never stalls its stream units on
// another warp's work. Entry: (row, sequence) for a row finalize, (sequence,
// slice) for a draw unit.
constexpr int kPend = 8;
struct Pending {
  int2* q;  // [kPend] this warp's ring in shared memory
  int head, n;
  __device__ __forceinline__ int2 front() const { return q[head]; }
  __device__ __forceinline__ void pop() {
    head = (head + 1) % kPend;
    --n;
  }
  __device__ __forceinline__ void push(int2 e) {
    WTRACE_ADD(4, 1);
    if ((threadIdx.x & 31) == 0) q[(head + n) % kPend] = e;
    __syncwarp();
    ++n;
  }
};

// Readiness probes: lane 0 issues a relaxed load of the task's count / flag
// early (its latency overlaps the stream unit); ready() reads it afterwards.
struct Probe {
  int v;
  __device__ __forceinline__ void issue(const int* p) {
    v = 0;
    if ((threadIdx.x & 31) == 0 && p) v = ld_relaxed(p);
  }
  __device__ __forceinline__ int value() {
    const int x = __shfl_sync(kFull, v, 0);
    __syncwarp();
    return x;
  }
};

template <typename T>
__device__ __forceinline__ void task_run(const PassArgs& p, bool draw, int2 e) {
  if (draw) pass_draw<T>(p, e.x, e.y);
  else pass_row<T>(p, e.x, e.y);
}

__device__ __forceinline__ const int* task_word(const PassArgs& p, bool draw, int2 e) {
  return draw ? p.pub + e.x : p.row_cnt + e.x;
}
__device__ __forceinline__ bool task_ok(const PassArgs& p, bool draw, int v) {
  return draw ? v != 0 : v >= p.fa.nsub;
}

// Blocking wait for a task's inputs (bug guard: DSDE_DERR_STALL after ~2 s).
__device__ __noinline__ bool task_wait(const PassArgs& p, bool draw, int2 e) {
#if DSDE_PASS_TRACE
  const unsigned long long t0 = gtimer();
#endif
  for (long long spin = 0; spin < (1LL << 22); ++spin) {
    Probe pr;
    pr.issue(task_word(p, draw, e));
    if (task_ok(p, draw, pr.value())) {
#if DSDE_PASS_TRACE
      WTRACE_ADD(3, gtimer() - t0);
#endif
      return true;
    }
    __nanosleep(spin < 64 ? 64 : 512);
  }
  if ((threadIdx.x & 31) == 0) raise_device_error(p.fa.err, DSDE_DERR_STALL, e.x);
  return false;
}

// One kind of task at the end of an iteration: the FIFO head if its probe
// says ready, then the newly attached task (run now if ready and nothing older
// waits, else queued; a full FIFO first waits for its oldest entry — its
// inputs belong to earlier iterations, pass.cuh header).
template <typename T>
__device__ __forceinline__ void tasks_step(const PassArgs& p, bool draw, Pending& f, Probe& head, bool has_new,
                                           int2 e, Probe& pe) {
  const int hv = head.value();
  const int nv = pe.value();
  if (f.n > 0 && task_ok(p, draw, hv)) {
    const int2 o = f.front();
    f.pop();
    task_run<T>(p, draw, o);
  }
  if (!has_new) return;
  if (f.n == 0 && task_ok(p, draw, nv)) {
    task_run<T>(p, draw, e);
    return;
  }
  if (f.n == kPend) {
    const int2 o = f.front();
    f.pop();
    if (task_wait(p, draw, o)) task_run<T>(p, draw, o);
  }
  f.push(e);
}

// Sequences that are malformed (k_i outside [1, DSDE_MAX_SL], rows outside the
// launch; every sequence when cu_sl is not a monotone prefix from 0) get
// accepted_len -1 and the device error here, by warp gw for i = gw, gw + W, ...;
// with dsde_step they also count towards the cap (SL^ = sl_min, state
// untouched), exactly as dsde_update_signal treats them.
__device__ __noinline__ void pass_invalid(const PassArgs& p, long long gw, long long W, bool all) {
  const FinArgs& a = p.fa;
  for (long long i = gw; i < a.B; i += W) {
    int c0, k;
    bool rows_ok = true;
    if (!all && seq_ok(a, (int)i, c0, k, &rows_ok)) continue;
    if ((threadIdx.x & 31) == 0) {
      a.acc_len[i] = -1;
      raise_device_error(a.err, rows_ok ? DSDE_DERR_BAD_SL : DSDE_DERR_ROWS, (int)i);
    }
    pass_signal(p, (int)i, 0, 0.0, -1);
  }
}

// measurement builds only: 1 = no finalize / draw tasks (the stream and its
// counts), 2 = also no counts, 3 = relaxed counts, 4 = draw units that only
// count (no weights), 5 = no draw tasks
#ifndef DSDE_PASS_EXP
#define DSDE_PASS_EXP 0
#endif
#ifndef DSDE_PASS_MINB
#define DSDE_PASS_MINB 3
#endif
constexpr int kPassThreads = 256;

template <typename T, bool ENT>
__global__ void __launch_bounds__(kPassThreads, ENT ? 2 : DSDE_PASS_MINB) k_pass(PassArgs p) {
  constexpr int NV = Traits<T>::NV;
  const FinArgs& a = p.fa;
  const long long W = (long long)gridDim.x * (kPassThreads / 32);
  const long long gw = (long long)blockIdx.x * (kPassThreads / 32) + (threadIdx.x >> 5);
#if DSDE_PASS_TRACE
  WTRACE_SET(0, gtimer());
  for (int k = 3; k < 8; ++k) WTRACE_SET(k, 0ull);
#endif
  // batch check (warp 0 of every CTA, while the other warps start streaming):
  // cu_sl must be a non-decreasing prefix from 0, else no row can be attributed
  // to a sequence and every sequence is a DSDE_DERR_BAD_SL error
  __shared__ volatile int s_state;  // 0 unknown, 1 ok, 2 malformed
  if (threadIdx.x == 0) s_state = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    int bad = __ldg(a.cu_sl) != 0;
#pragma unroll 8
    for (int i = threadIdx.x; i < a.B; i += 32) bad |= __ldg(a.cu_sl + i + 1) < __ldg(a.cu_sl + i);
    bad = __any_sync(kFull, bad);
    if (threadIdx.x == 0) s_state = bad ? 2 : 1;
  }
  auto malformed = [&]() -> bool {
    int v;
    while ((v = s_state) == 0) {
    }
    return v == 2;
  };
  // rows of this launch: sum k_i, or (device_rows) cu_sl[B] clamped to the capacity
  const int n_rows = a.dev_rows ? min(max(__ldg(a.cu_sl + a.B), 0), a.total) : a.total;
  const int nsub = a.nsub;
  const long long n_all = ((long long)n_rows + p.Ld) * nsub;
  long long q = gw;
  int r = (int)(q / nsub), u = (int)(q - (long long)r * nsub);
  const int dr = (int)(W / nsub), du = (int)(W - (long long)dr * nsub);
  int seq = 0, rseq = 0, dseq = 0;
  bool bad = false;
  __shared__ int2 s_pend[kPassThreads / 32][2][kPend];
  Pending rowq{s_pend[threadIdx.x >> 5][0], 0, 0}, drawq{s_pend[threadIdx.x >> 5][1], 0, 0};
  while (q < n_all) {
    // 1. readiness probes of the FIFO heads and of this iteration's attached
    //    tasks: (a) the row finalize (a2) of row r - Lr, attached to its slice
    //    (r - Lr) % nsub; (b) the draw unit (a4) of slice u of the sequence
    //    whose last row is r - Ld. Their loads are in flight during the stream unit.
    Probe rh, dh, rn, dn;
    rh.issue(rowq.n ? p.row_cnt + rowq.front().x : nullptr);
    dh.issue(drawq.n ? p.pub + drawq.front().x : nullptr);
    const int rr = r - p.Lr, rl = r - p.Ld;
    bool new_row = false, new_draw = false;
    if ((DSDE_PASS_EXP == 0 || DSDE_PASS_EXP >= 4) && rr >= 0 && rr < n_rows && u == rr % nsub) {
      rseq = seq_of_row(a.cu_sl, a.B, rseq, rr);
      new_row = true;
    }
    rn.issue(new_row ? p.row_cnt + rr : nullptr);
    if ((DSDE_PASS_EXP == 0 || DSDE_PASS_EXP == 4) && rl >= 0 && rl < n_rows) {
      dseq = seq_of_row(a.cu_sl, a.B, dseq, rl);
      int c0, k;
      new_draw = seq_ok(a, dseq, c0, k) && rl == c0 + k - 1;
    }
    dn.issue(new_draw ? p.pub + dseq : nullptr);
    // 2. stream unit (a1): the slice statistics, then count the slice in
    if (r < n_rows) {
      seq = seq_of_row(a.cu_sl, a.B, seq, r);
      uint4 rt[NV], rd[NV];
      load_slice<T>(reinterpret_cast<const T*>(a.tl) + (long long)(r + seq) * a.ld_t, a.V, u, rt);
      load_slice<T>(reinterpret_cast<const T*>(a.dl) + (long long)r * a.ld_d, a.V, u, rd);
      store_partial(const_cast<SubPartial*>(a.part) + ((long long)r * nsub + u),
                    slice_stats<T, NV, NoHook, ENT>(rt, rd));
      __syncwarp();
#if DSDE_PASS_EXP == 3
      if ((threadIdx.x & 31) == 0) atomicAdd(p.row_cnt + r, 1);
#elif DSDE_PASS_EXP != 2
      if ((threadIdx.x & 31) == 0) red_add_release(p.row_cnt + r, 1);
#endif
    }
    // 3. the finalize / draw work that is ready
    if (new_row || new_draw || rowq.n || drawq.n) {
      if ((bad = malformed())) break;
      tasks_step<T>(p, false, rowq, rh, new_row, make_int2(rr, rseq), rn);
      tasks_step<T>(p, true, drawq, dh, new_draw, make_int2(dseq, u), dn);
    }
    q += W;
    u += du;
    r += dr;
    if (u >= nsub) {
      u -= nsub;
      ++r;
    }
  }
#if DSDE_PASS_TRACE
  WTRACE_SET(1, gtimer());
#endif
  // the queued tasks (every stream unit of this warp is done; their inputs
  // come from earlier iterations of the other warps): whichever head is ready
  for (long long spin = 0; !bad && (rowq.n || drawq.n); ++spin) {
    Probe rh, dh;
    rh.issue(rowq.n ? p.row_cnt + rowq.front().x : nullptr);
    dh.issue(drawq.n ? p.pub + drawq.front().x : nullptr);
    const int rv = rh.value(), dv = dh.value();
    bool ran = false;
    if (rowq.n && task_ok(p, false, rv)) {
      const int2 o = rowq.front();
      rowq.pop();
      task_run<T>(p, false, o);
      ran = true;
    }
    if (drawq.n && task_ok(p, true, dv)) {
      const int2 o = drawq.front();
      drawq.pop();
      task_run<T>(p, true, o);
      ran = true;
    }
    if (ran) {
      spin = 0;
      continue;
    }
    if (spin > (1LL << 22)) {
      if ((threadIdx.x & 31) == 0) raise_device_error(a.err, DSDE_DERR_STALL, rowq.n ? rowq.front().x : drawq.front().x);
      break;
    }
    __nanosleep(spin < 64 ? 64 : 512);
  }
  pass_invalid(p, gw, W, bad || malformed());
#if DSDE_PASS_TRACE
  WTRACE_SET(2, gtimer());
#endif
}
