// state.cuh — layout of dsde_state (device side) and the verify workspace.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "dsde.h"

namespace dsde {

// Per-sequence adapter state (one slot per sequence), device resident.
// History ring of KLD observations (Fig.5): `count` valid values,
// the most recent at ring[(head - 1) mod n_long].
struct SeqState {
  double ring[DSDE_MAX_WINDOW];
  int head;
  int count;
  int steps;        // verification steps observed since reset
  int sl_a_max;     // Eq.1 SL_A,max over the calibration steps (D12)
  double kld_sum;   // Eq.1 numerator accumulators (mu_KLD,pre)
  long long kld_cnt;
  double kld_max;   // Eq.1 KLD_pre,max
  int sl_max;       // calibrated SL_max (Eq.1); 0 before calibration ends
  int calibrating;  // 1 while steps < calib_steps (set by update_signal)
  int last_sl_hat;
  int pad[3];
};
static_assert(sizeof(SeqState) % 16 == 0, "SeqState must stay 16-byte sized");

// Optional kernel timing of dsde_verify (dsde_profile_enable/read): events
// recorded before the first and after each launch of every call, reused
// across reads.
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // (DSDE_VERIFY_PHASES + 1) per recorded call
  size_t used = 0;
  cudaEvent_t next() {
    if (used == ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    return ev[used++];
  }
  ~Profiler() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

}  // namespace dsde

struct dsde_state_s {
  dsde_config cfg;
  int max_seqs;
  int device;
  dsde::SeqState* seq;   // [max_seqs]
  int32_t* err;          // [2]: code, sequence
  long long* scratch;    // [8]: cap partials (sum, n, max) for dsde_next_sl
  dsde::Profiler* prof;  // kernel timing (host side), created by dsde_profile_enable
  float* entropy_out;    // dsde_set_draft_entropy: H(q) per draft row, NULL = off
  const float* temps;    // dsde_set_temperature: T per sequence, NULL = 1 (D20)
};

struct dsde_comm_s {
  void* nccl;  // ncclComm_t
  int nranks, rank;
};
