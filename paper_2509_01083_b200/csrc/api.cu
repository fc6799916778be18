// api.cu — state lifetime, error word, and the NCCL communicator of the C-ABI.
//
// NCCL is resolved at run time with dlopen: in a PyTorch process the copy torch
// already loaded is reused (RTLD_NOLOAD), so the library never mixes two NCCL
// versions in one process; without a loaded copy it falls back to
// libnccl.so.2 on the loader path. Only the cap all-reduce (§8(e)) uses it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "common.cuh"
#include "state.cuh"

using namespace dsde;

namespace {

bool cfg_valid(const dsde_config& c) {
  return c.delta > 0.0 && c.delta <= 1.0 && c.n_short >= 1 && c.n_short < c.n_long &&
         c.n_long <= DSDE_MAX_WINDOW && c.sl_min >= 1 && c.sl_ceiling > c.sl_min &&
         c.sl_ceiling <= DSDE_MAX_SL && c.epsilon > 0.0 && c.calib_steps >= 0 &&
         c.calib_sl >= 1 && c.calib_sl <= c.sl_ceiling && (c.window_unit == 0 || c.window_unit == 1) &&
         (c.cap_mode == 0 || c.cap_mode == 1) && (c.greedy == 0 || c.greedy == 1) &&
         (c.device_rows == 0 || c.device_rows == 1) && (c.masked == 0 || c.masked == 1) &&
         (c.resample == DSDE_RESAMPLE_PROPOSAL || c.resample == DSDE_RESAMPLE_FULL) &&
         (c.entropy_mode == 0 || c.entropy_mode == 1) && c.entropy_gamma > 0.0;
}

__global__ void k_reset_slots(SeqState* seq, int max_seqs, const int32_t* slots, int n) {
  const int i = blockIdx.x;
  if (i >= n) return;
  const int s = slots[i];
  if (s < 0 || s >= max_seqs) return;
  uint4* p = reinterpret_cast<uint4*>(seq + s);
  for (int w = threadIdx.x; w < (int)(sizeof(SeqState) / 16); w += blockDim.x)
    p[w] = make_uint4(0, 0, 0, 0);
}

// ---- NCCL, resolved at run time ----
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.allReduce && api.allGather;
  });
  return api;
}

}  // namespace

// In-place int64 all-reduce of buf[0..n_sum) (sum) and, if max_at >= 0, of
// buf[max_at] (max) over the communicator, enqueued on stream s.
dsde_status dsde_comm_allreduce_i64(dsde_comm comm, long long* buf, int n_sum, int max_at,
                                    cudaStream_t s) {
  NcclApi& api = nccl();
  if (!api.ok || !comm) return DSDE_ERR_NCCL;
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm->nccl);
  if (api.allReduce(buf, buf, (size_t)n_sum, ncclInt64, ncclSum, c, s) != ncclSuccess)
    return DSDE_ERR_NCCL;
  if (max_at >= 0 &&
      api.allReduce(buf + max_at, buf + max_at, 1, ncclInt64, ncclMax, c, s) != ncclSuccess)
    return DSDE_ERR_NCCL;
  return DSDE_OK;
}

// The vocab-parallel exchanges (vocab.cuh): an in-place byte
// all-gather (each rank's block at recv + rank * bytes), a float sum and an
// int32 max all-reduce, enqueued on stream s.
dsde_status dsde_comm_allgather_bytes(dsde_comm comm, void* recv, size_t bytes, cudaStream_t s) {
  NcclApi& api = nccl();
  if (!api.ok || !comm) return DSDE_ERR_NCCL;
  ncclComm_t c = reinterpret_cast<ncclComm_t>(comm->nccl);
  const char* send = reinterpret_cast<const char*>(recv) + (size_t)comm->rank * bytes;
  return api.allGather(send, recv, bytes, ncclUint8, c, s) == ncclSuccess ? DSDE_OK : DSDE_ERR_NCCL;
}
dsde_status dsde_comm_allreduce_f32_sum(dsde_comm comm, float* buf, size_t n, cudaStream_t s) {
  NcclApi& api = nccl();
  if (!api.ok || !comm) return DSDE_ERR_NCCL;
  return api.allReduce(buf, buf, n, ncclFloat32, ncclSum, reinterpret_cast<ncclComm_t>(comm->nccl), s) ==
                 ncclSuccess ? DSDE_OK : DSDE_ERR_NCCL;
}
dsde_status dsde_comm_allreduce_i32_max(dsde_comm comm, int32_t* buf, size_t n, cudaStream_t s) {
  NcclApi& api = nccl();
  if (!api.ok || !comm) return DSDE_ERR_NCCL;
  return api.allReduce(buf, buf, n, ncclInt32, ncclMax, reinterpret_cast<ncclComm_t>(comm->nccl), s) ==
                 ncclSuccess ? DSDE_OK : DSDE_ERR_NCCL;
}
int dsde_comm_rank(dsde_comm comm) { return comm ? comm->rank : 0; }
int dsde_comm_size(dsde_comm comm) { return comm ? comm->nranks : 1; }

extern "C" {

void dsde_config_default(dsde_config* c) {
  if (!c) return;
  c->delta = 0.85;
  c->n_short = 10;
  c->n_long = 30;
  c->sl_min = 2;
  c->sl_ceiling = 8;
  c->epsilon = 1e-6;
  c->calib_steps = 5;
  c->calib_sl = 4;
  c->window_unit = 0;
  c->cap_mode = 1;
  c->greedy = 0;
  c->device_rows = 0;
  c->masked = 0;
  c->resample = DSDE_RESAMPLE_FULL;
  c->entropy_mode = 0;
  c->entropy_gamma = 0.5;
}

const char* dsde_status_string(dsde_status s) {
  switch (s) {
    case DSDE_OK: return "DSDE_OK";
    case DSDE_ERR_ARG: return "DSDE_ERR_ARG";
    case DSDE_ERR_CUDA: return "DSDE_ERR_CUDA";
    case DSDE_ERR_NCCL: return "DSDE_ERR_NCCL";
    case DSDE_ERR_STATE: return "DSDE_ERR_STATE";
    case DSDE_ERR_DEVICE: return "DSDE_ERR_DEVICE";
  }
  return "DSDE_UNKNOWN";
}

int dsde_abi_version(void) { return DSDE_ABI_VERSION; }

dsde_status dsde_state_create(const dsde_config* cfg, int max_seqs, dsde_state* out) {
  if (!cfg || !out || max_seqs < 1 || !cfg_valid(*cfg)) return DSDE_ERR_ARG;
  *out = nullptr;
  dsde_state st = static_cast<dsde_state>(calloc(1, sizeof(dsde_state_s)));
  if (!st) return DSDE_ERR_ARG;
  st->cfg = *cfg;
  st->max_seqs = max_seqs;
  cudaGetDevice(&st->device);
  const size_t seq_bytes = sizeof(SeqState) * (size_t)max_seqs;
  if (cudaMalloc(&st->seq, seq_bytes) != cudaSuccess ||
      cudaMalloc(&st->err, 2 * sizeof(int32_t)) != cudaSuccess ||
      cudaMalloc(&st->scratch, 8 * sizeof(long long)) != cudaSuccess ||
      cudaMemset(st->seq, 0, seq_bytes) != cudaSuccess ||
      cudaMemset(st->err, 0, 2 * sizeof(int32_t)) != cudaSuccess ||
      cudaMemset(st->scratch, 0, 8 * sizeof(long long)) != cudaSuccess ||
      cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(st->seq);
    cudaFree(st->err);
    cudaFree(st->scratch);
    free(st);
    return DSDE_ERR_CUDA;
  }
  *out = st;
  return DSDE_OK;
}

dsde_status dsde_state_reset(dsde_state st, const int32_t* slots, int n, void* stream) {
  if (!st || (!slots && n > 0) || n < 0) return DSDE_ERR_ARG;
  if (n == 0) return DSDE_OK;
  k_reset_slots<<<n, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(st->seq, st->max_seqs,
                                                                      slots, n);
  return cudaGetLastError() == cudaSuccess ? DSDE_OK : DSDE_ERR_CUDA;
}

dsde_status dsde_state_destroy(dsde_state st) {
  if (!st) return DSDE_OK;
  cudaDeviceSynchronize();
  cudaFree(st->seq);
  cudaFree(st->err);
  cudaFree(st->scratch);
  delete st->prof;
  free(st);
  return DSDE_OK;
}

dsde_status dsde_profile_enable(dsde_state st, int enable) {
  if (!st) return DSDE_ERR_ARG;
  if (!st->prof) st->prof = new dsde::Profiler();
  st->prof->on = enable != 0;
  return DSDE_OK;
}

dsde_status dsde_profile_read(dsde_state st, float* ms, int* calls) {
  if (!st || !ms) return DSDE_ERR_ARG;
  constexpr int P = DSDE_VERIFY_PHASES;
  for (int k = 0; k < P; ++k) ms[k] = 0.f;
  int n = 0;
  if (st->prof && st->prof->used > 0) {
    dsde::Profiler& pr = *st->prof;
    if (cudaEventSynchronize(pr.ev[pr.used - 1]) != cudaSuccess) return DSDE_ERR_CUDA;
    n = (int)(pr.used / (P + 1));
    for (int c = 0; c < n; ++c)
      for (int k = 0; k < P; ++k) {
        float t = 0.f;
        if (cudaEventElapsedTime(&t, pr.ev[c * (P + 1) + k], pr.ev[c * (P + 1) + k + 1]) != cudaSuccess)
          return DSDE_ERR_CUDA;
        ms[k] += t;
      }
    pr.used = 0;
  }
  if (calls) *calls = n;
  return DSDE_OK;
}

size_t dsde_state_bytes(dsde_state st) {
  return st ? sizeof(SeqState) * (size_t)st->max_seqs : 0;
}

dsde_status dsde_state_export(dsde_state st, void* buf, size_t bytes, void* stream) {
  if (!st || !buf || bytes < dsde_state_bytes(st)) return DSDE_ERR_ARG;
  return cudaMemcpyAsync(buf, st->seq, dsde_state_bytes(st), cudaMemcpyDeviceToDevice,
                         reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? DSDE_OK
             : DSDE_ERR_CUDA;
}

dsde_status dsde_state_import(dsde_state st, const void* buf, size_t bytes, void* stream) {
  if (!st || !buf || bytes < dsde_state_bytes(st)) return DSDE_ERR_ARG;
  return cudaMemcpyAsync(st->seq, buf, dsde_state_bytes(st), cudaMemcpyDeviceToDevice,
                         reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? DSDE_OK
             : DSDE_ERR_CUDA;
}

dsde_status dsde_get_device_error(dsde_state st, int32_t* code, int32_t* seq) {
  if (!st || !code || !seq) return DSDE_ERR_ARG;
  int32_t w[2] = {0, 0};
  if (cudaDeviceSynchronize() != cudaSuccess) return DSDE_ERR_CUDA;
  if (cudaMemcpy(w, st->err, sizeof(w), cudaMemcpyDeviceToHost) != cudaSuccess)
    return DSDE_ERR_CUDA;
  *code = w[0];
  *seq = w[0] ? w[1] : -1;
  return DSDE_OK;
}

dsde_status dsde_clear_device_error(dsde_state st, void* stream) {
  if (!st) return DSDE_ERR_ARG;
  return cudaMemsetAsync(st->err, 0, 2 * sizeof(int32_t),
                         reinterpret_cast<cudaStream_t>(stream)) == cudaSuccess
             ? DSDE_OK
             : DSDE_ERR_CUDA;
}

dsde_status dsde_comm_unique_id(uint8_t id[128]) {
  if (!id) return DSDE_ERR_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return DSDE_ERR_NCCL;
  ncclUniqueId u;
  if (api.getUniqueId(&u) != ncclSuccess) return DSDE_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  return DSDE_OK;
}

dsde_status dsde_comm_init(const uint8_t id[128], int nranks, int rank, dsde_comm* out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return DSDE_ERR_ARG;
  NcclApi& api = nccl();
  if (!api.ok) return DSDE_ERR_NCCL;
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ncclComm_t c = nullptr;
  if (api.commInitRank(&c, nranks, u, rank) != ncclSuccess) return DSDE_ERR_NCCL;
  dsde_comm cm = static_cast<dsde_comm>(calloc(1, sizeof(dsde_comm_s)));
  if (!cm) {
    api.commDestroy(c);
    return DSDE_ERR_ARG;
  }
  cm->nccl = c;
  cm->nranks = nranks;
  cm->rank = rank;
  *out = cm;
  return DSDE_OK;
}

dsde_status dsde_comm_destroy(dsde_comm comm) {
  if (!comm) return DSDE_OK;
  NcclApi& api = nccl();
  if (api.ok) api.commDestroy(reinterpret_cast<ncclComm_t>(comm->nccl));
  free(comm);
  return DSDE_OK;
}

}  // extern "C"
