// signal.cuh — per-sequence signal update (§8(a) a5-a6) and the cap helpers
// (a7), shared by signal.cu (dsde_update_signal / dsde_next_sl) and the fused
// step kernel in verify.cu (dsde_step).
//
// a5/a6: one warp per sequence. The KLD history is a per-slot fp64 ring of
// capacity n_long (Fig.5). Weighted variances (Eq.5-7):
// lanes hold the observations most recent first with alpha_i = delta^(i-1);
// the weighted mean and variance are two warp-wide fp64 reductions per window.
// a7: exact int64 partials (sum SL^, N, max SL^) -> optional NCCL all-reduce
// -> cap (Eq.11 with round-half-even, D14) -> next SL.
#pragma once

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
  const float* ent;  // [sum k] draft entropy per position (cfg.entropy_mode, D22), else NULL
};

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

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// One warp per sequence. Lane m holds history observations m and m + 32
// (most recent first, alpha = delta^m); the weighted mean and variance of
// Eq.6-7 are two warp-wide fp64 passes over the short and long windows.
// signal_seq_vals: the update from values in registers — lane j < k holds
// the fp32 KLD of position j (as a double), acc = a_i in every lane (-1: the
// verify flagged the sequence). signal_seq loads them from kld / acc_len.
// h: lane j < k holds the draft entropy of position j (entropy_mode, D22).
__device__ __forceinline__ void signal_seq_vals(const SignalArgs& a, int i, int k, double x, int acc,
                                                double h = 0.0) {
  const int lane = threadIdx.x & 31;
  const dsde_config& c = a.cfg;
  const int slot = a.slots[i];
  double* dg = a.diag ? a.diag + 8 * (long long)i : nullptr;
  if (slot < 0 || slot >= a.max_seqs) {
    if (lane == 0) {
      a.sl_hat[i] = c.sl_min;
      raise_device_error(a.err, DSDE_DERR_BAD_SLOT, i);
    }
    return;
  }
  SeqState& s = a.seq[slot];
  if (acc < 0 || k < 1 || k > DSDE_MAX_SL) {
    if (lane == 0) {
      a.sl_hat[i] = c.sl_min;  // verify flagged this sequence; its state is left untouched
      s.last_sl_hat = c.sl_min;
    }
    if (dg && lane < 8) dg[lane] = NAN;
    return;
  }
  if (lane >= k) x = 0.0;
  // 1-2: mu_last and the history append (Fig.5; D8)
  const double mu_last = wsum(x) / (double)k;
  const int cap = c.n_long;
  const int head0 = s.head, count0 = s.count;
  int n_new;
  if (c.window_unit == 0) {
    // oldest evicted by overwrite; if k > n_long only the last n_long are kept
    if (lane < k && lane >= k - cap) s.ring[(head0 + lane) % cap] = x;
    n_new = k;
  } else {
    if (lane == 0) s.ring[head0] = mu_last;
    n_new = 1;
  }
  const int head = (head0 + n_new) % cap;
  const int count = min(count0 + n_new, cap);
  // 3: calibration (Eq.1; D12)
  const int steps = s.steps + 1;
  const double ksum = wsum(x);
  double kmax = x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kmax = fmax(kmax, __shfl_xor_sync(kFull, kmax, o));
  int sl_max = s.sl_max;
  if (c.calib_steps < 1 && sl_max == 0) sl_max = c.sl_ceiling;
  int sl_a_max = s.sl_a_max;
  double kld_sum = s.kld_sum, kld_max = s.kld_max;
  long long kld_cnt = s.kld_cnt;
  if (steps <= c.calib_steps) {
    sl_a_max = max(sl_a_max, acc);
    kld_sum += ksum;
    kld_cnt += k;
    kld_max = fmax(kld_max, kmax);
    if (steps == c.calib_steps) sl_max = calib_sl_max(c, sl_a_max, kld_sum / (double)kld_cnt, kld_max);
  }
  __syncwarp();
  // 4-5: weighted variances (Eq.5-7) and WVIR (Eq.4; D9, D10)
  double var_s = NAN, var_l = NAN, wvir = 1.0;
  if (count >= c.n_short) {
    double xs[2], al[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = lane + 32 * h;  // m = 0 is the most recent observation
      xs[h] = m < count ? s.ring[(head - 1 - m + 2 * cap) % cap] : 0.0;
      al[h] = m < count ? pow(c.delta, (double)m) : 0.0;
    }
    double wv[2];
#pragma unroll
    for (int win = 0; win < 2; ++win) {
      const int N = win == 0 ? c.n_short : count;
      double sa = 0.0, sax = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = lane + 32 * h;
        if (m < N) {
          sa += al[h];
          sax += al[h] * xs[h];
        }
      }
      sa = wsum(sa);
      const double mu = wsum(sax) / sa;
      double sv = 0.0;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = lane + 32 * h;
        if (m < N) {
          const double e = xs[h] - mu;
          sv += al[h] * e * e;
        }
      }
      wv[win] = wsum(sv) / sa;
    }
    var_s = wv[0];
    var_l = wv[1];
    wvir = var_l < 1e-12 ? 1.0 : var_s / var_l;
  }
  // 6-7: SF (Eq.3), penalty and Eq.8
  const double sf = expm1(2.0 * mu_last);
  const double penalty = sf * wvir;
  const bool calibrating = steps < c.calib_steps;
  int out;
  double xr = NAN;
  if (calibrating) {
    out = c.calib_sl;
  } else {
    xr = penalty <= 1.0 ? (1.0 - penalty) * (double)(sl_max - c.sl_min) + (double)c.sl_min
                        : (double)c.sl_min;
    double rr = rint(xr);
    if (rr < c.sl_min) rr = c.sl_min;
    if (rr > sl_max) rr = sl_max;
    out = (int)rr;
    if (c.entropy_mode == 1 && a.ent) {
      // D22: SL_H from the mean draft entropy of the step, SL^ = min(SL^, SL_H)
      const double hm = wsum(lane < k ? h : 0.0) / (double)k;
      const double al = fmax(0.0, 1.0 - sqrt(c.entropy_gamma * hm));
      double rh = rint(al * (double)(sl_max - c.sl_min) + (double)c.sl_min);
      if (rh < c.sl_min) rh = c.sl_min;
      if (rh > sl_max) rh = sl_max;
      if ((int)rh < out) out = (int)rh;
    }
  }
  if (lane == 0) {
    s.head = head;
    s.count = count;
    s.steps = steps;
    s.sl_a_max = sl_a_max;
    s.kld_sum = kld_sum;
    s.kld_cnt = kld_cnt;
    s.kld_max = kld_max;
    s.sl_max = sl_max;
    s.calibrating = calibrating ? 1 : 0;
    s.last_sl_hat = out;
    a.sl_hat[i] = out;
  }
  if (dg && lane == 0) {
    dg[0] = mu_last;
    dg[1] = sf;
    dg[2] = var_s;
    dg[3] = var_l;
    dg[4] = wvir;
    dg[5] = penalty;
    dg[6] = xr;
    dg[7] = (double)sl_max;
  }
}

__device__ __forceinline__ void signal_seq(const SignalArgs& a, int i) {
  const int lane = threadIdx.x & 31;
  const int c0 = a.cu_sl[i], k = a.cu_sl[i + 1] - c0;
  const int acc = (c0 < 0 || k < 1 || k > DSDE_MAX_SL) ? -1 : a.acc_len[i];
  const double x = (acc >= 0 && lane < k) ? (double)a.kld[c0 + lane] : 0.0;
  const double h = (a.ent && acc >= 0 && lane < k) ? (double)a.ent[c0 + lane] : 0.0;
  signal_seq_vals(a, i, k, x, acc, h);
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

// L2 loads (ld.global.cg): in the fused step kernel these values were written
// by other CTAs of the same launch, so no L1 line may serve them.
__device__ __forceinline__ bool is_calibrating(const CapArgs& a, int i) {
  const int slot = __ldcg(a.slots + i);
  if (slot < 0 || slot >= a.max_seqs) return true;  // bad slot: excluded (error raised in signal)
  return __ldcg(&a.seq[slot].calibrating) != 0;
}

// Exact partial (sum, n, max) over the batch; one CTA, integer arithmetic.
__device__ __forceinline__ void cap_partial_block(const CapArgs& a, long long& sum, long long& n, long long& mx) {
  __shared__ long long s_v[3][32];
  long long ls = 0, ln = 0, lm = 0;
  for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
    if (is_calibrating(a, i)) continue;
    const long long v = __ldcg(a.sl_hat + i);
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

__device__ __forceinline__ void apply_cap(const CapArgs& a, int32_t cap) {
  for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
    const int sh = __ldcg(a.sl_hat + i);
    int v = is_calibrating(a, i) ? a.cfg.calib_sl : (sh < cap ? sh : cap);
    if (a.budget && a.budget[i] < v) v = a.budget[i];
    a.next_sl[i] = v;
  }
  if (threadIdx.x == 0) *a.cap = cap;
}

// a7 by one warp: exact int64 partial over the batch (lanes stride over
// sequences), the Eq.11 rule (D14), next SLs. Values written by other warps of
// this launch are read with ld.global.cg (is_calibrating / sl_hat).
__device__ __forceinline__ void cap_warp(const CapArgs& a) {
  const int lane = threadIdx.x & 31;
  long long ls = 0, ln = 0, lm = 0;
  for (int i = lane; i < a.B; i += 32) {
    if (is_calibrating(a, i)) continue;
    const long long v = __ldcg(a.sl_hat + i);
    ls += v;
    ln += 1;
    lm = v > lm ? v : lm;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ls += __shfl_xor_sync(kFull, ls, o);
    ln += __shfl_xor_sync(kFull, ln, o);
    const long long m2 = __shfl_xor_sync(kFull, lm, o);
    lm = m2 > lm ? m2 : lm;
  }
  const int32_t cap = cap_rule(a.cfg, ls, ln, lm);
  for (int i = lane; i < a.B; i += 32) {
    const int sh = __ldcg(a.sl_hat + i);
    int v = is_calibrating(a, i) ? a.cfg.calib_sl : (sh < cap ? sh : cap);
    if (a.budget && a.budget[i] < v) v = a.budget[i];
    a.next_sl[i] = v;
  }
  if (lane == 0) *a.cap = cap;
}

}  // namespace dsde
