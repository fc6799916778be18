// pipe_bench.cu — per-SM throughput of the instruction classes the stream
// kernel is built from (B200 measurements for DESIGN.md §6):
//   MUFU.EX2 (ex2.approx.ftz.f32), FFMA2 (packed fp32 FMA), FFMA, DFMA,
//   PRMT/LOP3 (ALU), and a mixed FFMA2 + MUFU stream.
// Each thread runs 8 independent chains so latency is hidden; the grid fills
// every SM with 32 warps. Reported as lane-operations per clock per SM.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void k_mufu(float* out, float s) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = s * (threadIdx.x + j) * 1e-6f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = ex2(a[j]) * -0.5f;
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_mufu_only(float* out, float s) {  // ex2 chains without the FMUL
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = -s * (threadIdx.x + j) * 1e-6f;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = -ex2(a[j]);
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_ffma2(float* out, float s) {
  float2 a[8];
  const float2 m = make_float2(0.999f, 0.998f), c = make_float2(s, s);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = make_float2(threadIdx.x + j, j);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __ffma2_rn(a[j], m, c);
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j].x + a[j].y;
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_ffma2_reg(float* out, float s, float s2) {  // all-register operands
  float2 a[8];
  const float2 m = make_float2(s2, s2 * 0.5f), c = make_float2(s, s * 2.f);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = make_float2(threadIdx.x + j, j);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __ffma2_rn(a[j], m, c);
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j].x + a[j].y;
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_ffma(float* out, float s, float s2) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], s2, s);
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == 1234.5f) out[0] = r;
}

__global__ void k_dfma(float* out, double s, double s2) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], s2, s);
  }
  double r = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += a[j];
  if (r == 1234.5) out[0] = (float)r;
}

__global__ void k_alu(float* out, unsigned s) {
  unsigned a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 7 + j;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __byte_perm(a[j], s, 0x1044) ^ (a[j] & 0xffff0000u);
  }
  unsigned r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= a[j];
  if (r == 12345u) out[0] = (float)r;
}

// 2 MUFU + 10 FFMA2 per step (the stream kernel's ratio, roughly)
__global__ void k_mix(float* out, float s) {
  float2 a[4];
  const float2 m = make_float2(0.999f, 0.998f), c = make_float2(s, s);
#pragma unroll
  for (int j = 0; j < 4; ++j) a[j] = make_float2((threadIdx.x + j) * 1e-6f, j * 1e-6f);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float2 e = make_float2(ex2(-a[j].x), ex2(-a[j].y));
#pragma unroll
      for (int k = 0; k < 10; ++k) e = __ffma2_rn(e, m, c);
      a[j] = __fmul2_rn(e, make_float2(1e-3f, 1e-3f));
    }
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) r += a[j].x + a[j].y;
  if (r == 1234.5f) out[0] = r;
}

template <typename F>
void run(const char* name, F launch, double lane_ops_per_thread, int sms, int clk_khz) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double threads = (double)sms * 4 * 256;  // grid below: sms * 4 blocks of 256 threads
  const double ops = threads * lane_ops_per_thread;
  const double per_clk_sm = ops / (ms * 1e-3) / (clk_khz * 1e3) / sms;
  printf("%-12s %8.3f ms  %8.1f lane-ops/clk/SM  (%s)\n", name, ms, per_clk_sm, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d, clock %d kHz\n", sms, clk);
  float* out;
  cudaMalloc(&out, 4);
  const dim3 g(sms * 4), b(256);  // 32 warps per SM
  run("mufu+fmul", [&] { k_mufu<<<g, b>>>(out, 1.f); }, ITERS * 8.0, sms, clk);
  run("mufu", [&] { k_mufu_only<<<g, b>>>(out, 1.f); }, ITERS * 8.0, sms, clk);
  run("ffma2(imm)", [&] { k_ffma2<<<g, b>>>(out, 1.f); }, ITERS * 16.0, sms, clk);
  run("ffma2(reg)", [&] { k_ffma2_reg<<<g, b>>>(out, 1.f, 0.999f); }, ITERS * 16.0, sms, clk);
  run("ffma", [&] { k_ffma<<<g, b>>>(out, 1.f, 0.999f); }, ITERS * 8.0, sms, clk);
  run("dfma", [&] { k_dfma<<<g, b>>>(out, 1.0, 0.999); }, ITERS * 8.0, sms, clk);
  run("prmt+lop3", [&] { k_alu<<<g, b>>>(out, 7u); }, ITERS * 8.0 * 2, sms, clk);
  run("mix 2mufu+10ffma2 (mufu lane-ops)", [&] { k_mix<<<g, b>>>(out, 1.f); }, ITERS * 4.0 * 2, sms, clk);
  return 0;
}
