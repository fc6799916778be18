// signal.cu — dsde_update_signal (§8(a) a5-a6) and dsde_next_sl (a7); the
// per-sequence and cap device code is in signal.cuh.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "common.cuh"
#include "state.cuh"
#include "signal.cuh"

// Implemented in api.cu (NCCL resolved at run time).
dsde_status dsde_comm_allreduce_i64(dsde_comm comm, long long* buf, int n_sum, int max_at,
                                    cudaStream_t s);

namespace dsde {

__global__ void __launch_bounds__(128) k_update_signal(SignalArgs a) {
  const int i = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (i >= a.B) return;
  signal_seq(a, i);
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

// Multi-GPU cap: exact partial -> NCCL all-reduce (sum; + max for cap_mode 0)
// -> cap and next SL, enqueued on s. *st receives DSDE_ERR_NCCL on failure.
cudaError_t launch_cap_multi(const CapArgs& a, dsde_comm comm, cudaStream_t s, dsde_status* st) {
  *st = DSDE_OK;
  k_cap_partial<<<1, 1024, 0, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  *st = dsde_comm_allreduce_i64(comm, a.scratch, 2, a.cfg.cap_mode == 0 ? 2 : -1, s);
  if (*st != DSDE_OK) return cudaSuccess;
  k_cap_apply<<<1, 1024, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace dsde

using namespace dsde;


extern "C" int32_t dsde_cap_value(const dsde_config* cfg, int64_t sum_sl_hat, int64_t n_active,
                                  int64_t max_sl_hat) {
  if (!cfg) return -1;
  return cap_rule(*cfg, sum_sl_hat, n_active, max_sl_hat);
}

extern "C" dsde_status dsde_update_signal(dsde_state st, int B, const int32_t* slots,
                                          const int32_t* cu_sl, const float* kld,
                                          const int32_t* accepted_len, int32_t* sl_hat,
                                          double* diag, void* stream) {
  NvtxRange nv("dsde_update_signal");
  if (!st || !slots || !cu_sl || !kld || !accepted_len || !sl_hat || B < 1) return DSDE_ERR_ARG;
  if (B > st->max_seqs) return DSDE_ERR_STATE;
  if (st->cfg.entropy_mode && !st->entropy_out) return DSDE_ERR_ARG;  // D22 reads the draft entropy
  SignalArgs a{st->cfg, B, st->max_seqs, slots, cu_sl, kld, accepted_len, sl_hat, diag, st->seq,
               st->err, st->cfg.entropy_mode ? st->entropy_out : nullptr};
  k_update_signal<<<(B + 3) / 4, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a);
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

extern "C" dsde_status dsde_next_sl(dsde_state st, int B, const int32_t* slots,
                                    const int32_t* sl_hat, const int32_t* budget,
                                    int32_t* next_sl, int32_t* cap, dsde_comm comm,
                                    void* stream) {
  NvtxRange nv("dsde_next_sl");
  if (!st || !slots || !sl_hat || !next_sl || !cap || B < 1) return DSDE_ERR_ARG;
  if (B > st->max_seqs) return DSDE_ERR_STATE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  CapArgs a{st->cfg, B, st->max_seqs, slots, sl_hat, budget, next_sl, cap, st->seq, st->scratch};
  if (!comm) {
    k_cap_local<<<1, 1024, 0, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
  }
  dsde_status rs = DSDE_OK;
  const cudaError_t e = launch_cap_multi(a, comm, s, &rs);
  if (rs != DSDE_OK) return rs;
  return e == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}
