// tma_stream_bench.cu — microbenchmark: how fast can a persistent kernel stream
// a large buffer from HBM with 1-D TMA bulk copies into a shared-memory ring
// (the memory side of k_stream_ws), as a function of stage size, stage count
// and CTAs per SM. Consumers only touch one word per 16 bytes (LDS.128) and
// release the stage. Also times a plain LDG.128 streaming kernel for reference.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream_bench tma_stream_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nLW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n@P1 bra DN;\nbra LW;\nDN:\n}\n" ::"r"(sa(b)),
               "r"(par), "r"(0x100000u) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}

template <int STAGE, int NST, int CW>
__global__ void k_tma(const uint8_t* src, long long n_items, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)(sm + NST * STAGE);
  uint64_t* cons = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&cons[s], CW); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == CW) {
    if (lane == 0) {
      long long q = blockIdx.x;
      for (int s = 0; s < NST && q < n_items; ++s, q += G) {
        mbar_expect(&full[s], STAGE);
        bulk(sm + s * STAGE, src + q * STAGE, STAGE, &full[s]);
      }
      int s = 0; unsigned rnd = 0;
      for (; q < n_items; q += G) {
        mbar_wait(&cons[s], rnd & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect(&full[s], STAGE);
        bulk(sm + s * STAGE, src + q * STAGE, STAGE, &full[s]);
        if (++s == NST) { s = 0; ++rnd; }
      }
    }
    return;
  }
  unsigned acc = 0;
  int s = 0; unsigned rnd = 0;
  for (long long q = blockIdx.x; q < n_items; q += G) {
    mbar_wait(&full[s], rnd & 1);
    const uint4* p = (const uint4*)(sm + s * STAGE);
    for (int i = warp * 32 + lane; i < STAGE / 16; i += CW * 32) { uint4 v = p[i]; acc ^= v.x ^ v.w; }
    __syncwarp();
    if (lane == 0) mbar_arrive(&cons[s]);
    if (++s == NST) { s = 0; ++rnd; }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void k_ldg(const uint4* src, long long n16, unsigned* sink) {
  unsigned acc = 0;
  long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n16; i += stride) acc ^= __ldcs(src + i).x;
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int STAGE, int NST, int CW>
void run(const uint8_t* buf, size_t bytes, unsigned* sink, int ctas_per_sm, int sms) {
  const int smem = NST * STAGE + 2 * NST * 8;
  cudaFuncSetAttribute(k_tma<STAGE, NST, CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long items = bytes / STAGE;
  int grid = sms * ctas_per_sm;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) k_tma<STAGE, NST, CW><<<grid, 32 * (CW + 1), smem>>>(buf, items, sink);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int w = 0; w < reps; ++w) k_tma<STAGE, NST, CW><<<grid, 32 * (CW + 1), smem>>>(buf, items, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  printf("tma stage=%6d stages=%d cwarps=%2d ctas/sm=%d smem=%6d : %7.1f GB/s %s\n", STAGE, NST, CW, ctas_per_sm, smem,
         items * (double)STAGE * reps / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 4ull << 30;
  uint8_t* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
  unsigned* sink; cudaMalloc(&sink, 4);
  {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int bs : {256, 512}) for (int g : {1, 2, 4, 8}) {
      k_ldg<<<sms * g, bs>>>((const uint4*)buf, bytes / 16, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_ldg<<<sms * g, bs>>>((const uint4*)buf, bytes / 16, sink);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("ldg  block=%d grid=%d x SMs : %7.1f GB/s\n", bs, g, bytes * 5.0 / (ms * 1e-3) / 1e9);
    }
  }
  run<32768, 3, 8>(buf, bytes, sink, 2, sms);
  run<32768, 3, 8>(buf, bytes, sink, 1, sms);
  run<32768, 6, 8>(buf, bytes, sink, 1, sms);
  run<16384, 6, 8>(buf, bytes, sink, 2, sms);
  run<16384, 4, 8>(buf, bytes, sink, 2, sms);
  run<16384, 3, 4>(buf, bytes, sink, 4, sms);
  run<8192, 6, 4>(buf, bytes, sink, 4, sms);
  run<65536, 3, 8>(buf, bytes, sink, 1, sms);
  run<32768, 2, 8>(buf, bytes, sink, 3, sms);
  return 0;
}
