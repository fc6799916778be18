// common.cuh — device helpers shared by the DSDE kernels (product path only).
//
// Nothing here is shared with oracle/: the oracle is an independent C
// program. Citation keys as in include/dsde.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dsde.h"
#include <nvtx3/nvToolsExt.h>

namespace dsde {

// NVTX range over a host API call (a no-op unless a profiler is attached):
// the call's kernel launches appear under the entry point's name in
// Nsight Systems / ncu --nvtx.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
constexpr double kLn2d = 0.6931471805599453094;
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11) keyed by a 64-bit seed, counter 0, and
// the res53 map to doubles in [0,1) (D6): words 0-1 -> u_acc, 2-3 -> u_smp.
// ---------------------------------------------------------------------------
struct Uniforms {
  double acc, smp;
};

// ctr0: the counter's first word — 0 for D6's (u_acc, u_smp); j >= 1 for the
// (u_prop, u_keep) of recovery-draw proposal j (D23).
__device__ __forceinline__ Uniforms philox_uniforms(uint64_t seed, uint32_t ctr0 = 0u) {
  uint32_t c0 = ctr0, c1 = 0u, c2 = 0u, c3 = 0u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  Uniforms u;
  u.acc = ((double)(c0 >> 5) * 67108864.0 + (double)(c1 >> 6)) * 0x1.0p-53;
  u.smp = ((double)(c2 >> 5) * 67108864.0 + (double)(c3 >> 6)) * 0x1.0p-53;
  return u;
}

// ex2.approx (MUFU.EX2): 2^x with ~2 ulp relative error; flushes denormals.
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// bf16 pair in a 32-bit word -> two exact fp32 values.
// (byte permutes run on the ALU pipe; a plain shift is often lowered to IMAD,
// which competes with the FFMA2 stream on the FMA pipe)
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(__byte_perm(w, 0u, 0x1044)); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) {
  return __uint_as_float((uint32_t)b << 16);
}

template <typename T>
__device__ __forceinline__ float load_logit(const T* p);
template <>
__device__ __forceinline__ float load_logit<float>(const float* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float load_logit<uint16_t>(const uint16_t* p) {
  return bf16_bits_to_float(__ldg(p));
}

// 128-bit streaming load that does not allocate in L1 (read-once data).
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Sticky device error word: the first error wins (code, sequence index).
__device__ __forceinline__ void raise_device_error(int32_t* word, int code, int seq) {
  if (word == nullptr) return;
  if (atomicCAS(word, 0, code) == 0) atomicExch(word + 1, seq);
}

}  // namespace dsde
