// microbench.cu -- measured on-chip peaks for the roofline of the gather
// kernels (bench.py "roofline"): FP32 FMA-pipe throughput (FFMA and the
// paired FFMA2 of fma.rn.f32x2) and the L2 read bandwidth of 256-bit
// L1::no_allocate loads from an L2-resident buffer (the FP's cell loads).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
//   ./microbench > profiles/r02_microbench.json
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void ffma_kernel(float* out, float a, float b) {
  float x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fmaf(x[c], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, float a, float b) {
  unsigned long long x[CHAINS / 2], A, B;
  asm("mov.b64 %0, {%1, %1};" : "=l"(A) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(B) : "f"(b));
#pragma unroll
  for (int c = 0; c < CHAINS / 2; ++c) {
    float lo = threadIdx.x * 1e-3f + c, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[c]) : "f"(lo), "f"(hi));
  }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS / 2; ++c)
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS / 2; ++c) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[c]));
    s += lo + hi;
  }
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// every warp streams the whole L2-resident buffer (32-byte sectors, 256-bit
// loads, no L1 allocation), starting at a warp-dependent offset
__global__ void l2_read_kernel(const float4* __restrict__ buf, size_t n_cells, int passes,
                               float* out) {
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  size_t i = (warp * 7919u * 32u + lane) % n_cells;
  float acc = 0.f;
  for (int p = 0; p < passes; ++p) {
#pragma unroll 8
    for (int k = 0; k < 64; ++k) {
      float a0, a1, a2, a3, a4, a5, a6, a7;
      asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6),
                     "=f"(a7)
                   : "l"(buf + 2 * i));
      acc += (a0 + a1) + (a2 + a3) + (a4 + a5) + (a6 + a7);
      i += 32;
      if (i >= n_cells) i -= n_cells;
    }
  }
  if (acc == 1234.5f) out[0] = acc;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  float* out;
  CK(cudaMalloc(&out, 4096 * sizeof(float)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);

  // FMA pipe: blocks of 256 threads, 8 per SM, many waves
  const int blocks = sms * 8 * 16, threads = 256;
  double best_ffma = 0, best_ffma2 = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    double lane_fma = (double)blocks * threads * ITERS * CHAINS;
    double v = lane_fma / (time_ms(e0, e1) * 1e-3);
    if (v > best_ffma) best_ffma = v;
    cudaEventRecord(e0);
    ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    v = lane_fma / (time_ms(e0, e1) * 1e-3);
    if (v > best_ffma2) best_ffma2 = v;
  }

  // L2 read: 48 MiB buffer (well inside the 126 MB L2), warmed first
  const size_t bytes = 48ull << 20, cells = bytes / 32;
  float4* buf;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 0, bytes));
  const int lblocks = sms * 8, lthreads = 256, passes = 64;
  l2_read_kernel<<<lblocks, lthreads>>>(buf, cells, 4, out);
  double best_l2 = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    l2_read_kernel<<<lblocks, lthreads>>>(buf, cells, passes, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    double b = (double)lblocks * lthreads * passes * 64 * 32;
    double v = b / (time_ms(e0, e1) * 1e-3);
    if (v > best_l2) best_l2 = v;
  }
  CK(cudaGetLastError());
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_rate_mhz_attr\": %.0f,\n", prop.name, sms,
         clk_khz / 1e3);
  printf(" \"ffma_lane_fma_per_s\": %.6e, \"ffma2_lane_fma_per_s\": %.6e,\n", best_ffma,
         best_ffma2);
  printf(" \"fp32_tflops_ffma\": %.2f, \"fp32_tflops_ffma2\": %.2f,\n", 2 * best_ffma / 1e12,
         2 * best_ffma2 / 1e12);
  printf(" \"l2_read_gbs\": %.1f, \"l2_read_buffer_mib\": %zu,\n", best_l2 / 1e9, bytes >> 20);
  printf(" \"how\": \"best of 5 CUDA-event-timed launches; FMA: %d blocks x %d threads x %d "
         "iterations x %d independent chains (FFMA2: fma.rn.f32x2, 2 lane-FMAs each); L2: every "
         "warp streams a %zu MiB L2-resident buffer with ld.global.nc.L1::no_allocate.v8.f32 "
         "(one 32-byte sector per lane)\"}\n",
         blocks, threads, ITERS, CHAINS, bytes >> 20);
  return 0;
}
