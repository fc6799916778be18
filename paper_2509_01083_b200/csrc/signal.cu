// signal.cu — dsde_update_signal (§8(a) a5-a6) and dsde_next_sl (a7).
//
// a5/a6: one thread per sequence. The KLD history is a per-slot fp64 ring of
// capacity n_long (Fig.5). Weighted variances (Eq.5-7)
// use West's weighted incremental recurrence (CACM 22(9), 1979) over the ring,
// most recent observation first (alpha_1 = 1), snapshotting the short window
// on the way to the long one — one pass, no second sweep.
// a7: exact int64 partials (sum SL^, N, max SL^) -> optional NCCL all-reduce
// -> cap (Eq.11 with round-half-even, D14) -> next SL.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "state.cuh"

namespace dsde {

struct SignalArgs {
  dsde_config cfg;
  int B;
  int max_seqs;
  const int32_t* slots;
  const int32_t* cu_sl;
  const float* kld;
  const int32_t* acc_len;
  int32_t* sl_hat;
  double* diag;
  SeqState* seq;
  int32_t* err;
};

__device__ __forceinline__ void ring_push(SeqState& s, int cap, double x) {
  s.ring[s.head] = x;
  s.head = s.head + 1 == cap ? 0 : s.head + 1;
  if (s.count < cap) s.count++;
}

// Eq.1 + D11: SL_max = clamp(rint(raw), sl_min + 1, sl_ceiling).
__host__ __device__ inline int calib_sl_max(const dsde_config& c, int sl_a_max, double mu,
                                            double mx) {
  if (sl_a_max <= 0) return c.sl_min + 1;
  const double raw = (double)sl_a_max * (1.0 + mu / (mx + c.epsilon));
  double r = rint(raw);
  if (r < c.sl_min + 1) r = c.sl_min + 1;
  if (r > c.sl_ceiling) r = c.sl_ceiling;
  return (int)r;
}

__global__ void k_update_signal(SignalArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.B) return;
  const dsde_config& c = a.cfg;
  const int slot = a.slots[i];
  double* dg = a.diag ? a.diag + 8 * (long long)i : nullptr;
  if (slot < 0 || slot >= a.max_seqs) {
    a.sl_hat[i] = c.sl_min;
    raise_device_error(a.err, DSDE_DERR_BAD_SLOT, i);
    return;
  }
  SeqState& s = a.seq[slot];
  const int c0 = a.cu_sl[i], k = a.cu_sl[i + 1] - c0;
  if (a.acc_len[i] < 0 || k < 1 || k > DSDE_MAX_SL || c0 < 0) {
    a.sl_hat[i] = c.sl_min;  // verify flagged this sequence; leave its state untouched
    s.last_sl_hat = c.sl_min;
    if (dg)
      for (int q = 0; q < 8; ++q) dg[q] = NAN;
    return;
  }
  // 1-2: mu_last and history append (D8: per-token or per-step unit)
  double sum = 0.0;
  for (int j = 0; j < k; ++j) sum += (double)a.kld[c0 + j];
  const double mu_last = sum / (double)k;
  if (c.window_unit == 0) {
    for (int j = 0; j < k; ++j) ring_push(s, c.n_long, (double)a.kld[c0 + j]);
  } else {
    ring_push(s, c.n_long, mu_last);
  }
  s.steps++;
  // 3: calibration (Eq.1; D12)
  if (c.calib_steps < 1 && s.sl_max == 0) s.sl_max = c.sl_ceiling;
  if (s.steps <= c.calib_steps) {
    if (a.acc_len[i] > s.sl_a_max) s.sl_a_max = a.acc_len[i];
    for (int j = 0; j < k; ++j) {
      const double x = (double)a.kld[c0 + j];
      s.kld_sum += x;
      s.kld_cnt += 1;
      if (x > s.kld_max) s.kld_max = x;
    }
    if (s.steps == c.calib_steps)
      s.sl_max = calib_sl_max(c, s.sl_a_max, s.kld_sum / (double)s.kld_cnt, s.kld_max);
  }
  // 4-5: weighted variances, most recent first, and WVIR (Eq.4; D9, D10)
  double var_s = NAN, var_l = NAN, wvir = 1.0;
  if (s.count >= c.n_short) {
    double W = 0.0, mean = 0.0, S2 = 0.0, alpha = 1.0;
    int pos = s.head;
    for (int n = 1; n <= s.count; ++n) {
      pos = pos == 0 ? c.n_long - 1 : pos - 1;
      const double x = s.ring[pos];
      const double Wn = W + alpha;
      const double q = x - mean;
      const double r = q * alpha / Wn;
      mean += r;
      S2 += W * q * r;
      W = Wn;
      alpha *= c.delta;
      if (n == c.n_short) var_s = S2 / W;
    }
    var_l = S2 / W;
    wvir = var_l < 1e-12 ? 1.0 : var_s / var_l;
  }
  // 6-7: SF (Eq.3), penalty and Eq.8
  const double sf = expm1(2.0 * mu_last);
  const double penalty = sf * wvir;
  const bool calibrating = s.steps < c.calib_steps;
  int out;
  double x = NAN;
  if (calibrating) {
    out = c.calib_sl;
  } else {
    x = penalty <= 1.0 ? (1.0 - penalty) * (double)(s.sl_max - c.sl_min) + (double)c.sl_min
                       : (double)c.sl_min;
    double rr = rint(x);
    if (rr < c.sl_min) rr = c.sl_min;
    if (rr > s.sl_max) rr = s.sl_max;
    out = (int)rr;
  }
  s.calibrating = calibrating ? 1 : 0;
  s.last_sl_hat = out;
  a.sl_hat[i] = out;
  if (dg) {
    dg[0] = mu_last;
    dg[1] = sf;
    dg[2] = var_s;
    dg[3] = var_l;
    dg[4] = wvir;
    dg[5] = penalty;
    dg[6] = x;
    dg[7] = (double)s.sl_max;
  }
}

// Eq.11 integerised exactly (D14): q, r = divmod(sum, n); round half
// to even. cap_mode 0: the max (no cap). n == 0: sl_ceiling.
__host__ __device__ inline int32_t cap_rule(const dsde_config& c, long long sum, long long n,
                                            long long mx) {
  if (n <= 0) return c.sl_ceiling;
  if (c.cap_mode == 0) return (int32_t)mx;
  long long q = sum / n, r = sum % n;
  if (2 * r > n || (2 * r == n && (q & 1))) q += 1;
  return (int32_t)q;
}

struct CapArgs {
  dsde_config cfg;
  int B, max_seqs;
  const int32_t* slots;
  const int32_t* sl_hat;
  const int32_t* budget;
  int32_t* next_sl;
  int32_t* cap;
  const SeqState* seq;
  long long* scratch;  // [0] sum, [1] n, [2] max (all-reduced in place)
};

__device__ __forceinline__ bool is_calibrating(const CapArgs& a, int i) {
  const int slot = a.slots[i];
  if (slot < 0 || slot >= a.max_seqs) return true;  // bad slot: excluded (error raised in signal)
  return a.seq[slot].calibrating != 0;
}

// Exact partial (sum, n, max) over the batch; one CTA, integer arithmetic.
__device__ void cap_partial_block(const CapArgs& a, long long& sum, long long& n, long long& mx) {
  __shared__ long long s_v[3][32];
  long long ls = 0, ln = 0, lm = 0;
  for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
    if (is_calibrating(a, i)) continue;
    const long long v = a.sl_hat[i];
    ls += v;
    ln += 1;
    lm = v > lm ? v : lm;
  }
  for (int o = 16; o > 0; o >>= 1) {
    ls += __shfl_xor_sync(kFull, ls, o);
    ln += __shfl_xor_sync(kFull, ln, o);
    const long long m2 = __shfl_xor_sync(kFull, lm, o);
    lm = m2 > lm ? m2 : lm;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s_v[0][warp] = ls;
    s_v[1][warp] = ln;
    s_v[2][warp] = lm;
  }
  __syncthreads();
  sum = 0;
  n = 0;
  mx = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    sum += s_v[0][w];
    n += s_v[1][w];
    mx = s_v[2][w] > mx ? s_v[2][w] : mx;
  }
}

__device__ void apply_cap(const CapArgs& a, int32_t cap) {
  for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
    int v = is_calibrating(a, i) ? a.cfg.calib_sl : (a.sl_hat[i] < cap ? a.sl_hat[i] : cap);
    if (a.budget && a.budget[i] < v) v = a.budget[i];
    a.next_sl[i] = v;
  }
  if (threadIdx.x == 0) *a.cap = cap;
}

// Single GPU: partial -> cap -> next SL in one launch.
__global__ void __launch_bounds__(1024) k_cap_local(CapArgs a) {
  long long s, n, m;
  cap_partial_block(a, s, n, m);
  apply_cap(a, cap_rule(a.cfg, s, n, m));
}

// Multi-GPU: partial to scratch, all-reduce (host enqueues NCCL), then apply.
__global__ void __launch_bounds__(1024) k_cap_partial(CapArgs a) {
  long long s, n, m;
  cap_partial_block(a, s, n, m);
  if (threadIdx.x == 0) {
    a.scratch[0] = s;
    a.scratch[1] = n;
    a.scratch[2] = m;
  }
}

__global__ void __launch_bounds__(1024) k_cap_apply(CapArgs a) {
  apply_cap(a, cap_rule(a.cfg, a.scratch[0], a.scratch[1], a.scratch[2]));
}

}  // namespace dsde

using namespace dsde;

// Implemented in api.cu (NCCL resolved at run time).
dsde_status dsde_comm_allreduce_i64(dsde_comm comm, long long* buf, int n_sum, int max_at,
                                    cudaStream_t s);

extern "C" int32_t dsde_cap_value(const dsde_config* cfg, int64_t sum_sl_hat, int64_t n_active,
                                  int64_t max_sl_hat) {
  if (!cfg) return -1;
  return cap_rule(*cfg, sum_sl_hat, n_active, max_sl_hat);
}

extern "C" dsde_status dsde_update_signal(dsde_state st, int B, const int32_t* slots,
                                          const int32_t* cu_sl, const float* kld,
                                          const int32_t* accepted_len, int32_t* sl_hat,
                                          double* diag, void* stream) {
  if (!st || !slots || !cu_sl || !kld || !accepted_len || !sl_hat || B < 1) return DSDE_ERR_ARG;
  if (B > st->max_seqs) return DSDE_ERR_STATE;
  SignalArgs a{st->cfg, B, st->max_seqs, slots, cu_sl, kld, accepted_len, sl_hat, diag, st->seq,
               st->err};
  k_update_signal<<<(B + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

extern "C" dsde_status dsde_next_sl(dsde_state st, int B, const int32_t* slots,
                                    const int32_t* sl_hat, const int32_t* budget,
                                    int32_t* next_sl, int32_t* cap, dsde_comm comm,
                                    void* stream) {
  if (!st || !slots || !sl_hat || !next_sl || !cap || B < 1) return DSDE_ERR_ARG;
  if (B > st->max_seqs) return DSDE_ERR_STATE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CapArgs a{st->cfg, B, st->max_seqs, slots, sl_hat, budget, next_sl, cap, st->seq, st->scratch};
  if (!comm) {
    k_cap_local<<<1, 1024, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
  }
  k_cap_partial<<<1, 1024, 0, s>>>(a);
  if (cudaGetLastError() != cudaSuccess) return DSDE_ERR_CUDA;
  const dsde_status r =
      dsde_comm_allreduce_i64(comm, st->scratch, 2, st->cfg.cap_mode == 0 ? 2 : -1, s);
  if (r != DSDE_OK) return r;
  k_cap_apply<<<1, 1024, 0, s>>>(a);
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}
