// l1_wavefronts.cu -- how many L1TEX data-pipe wavefronts a warp-wide global
// load costs, as a function of the access pattern (run under ncu with
// --metrics l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,
//            l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum).
// Each kernel issues ITERS loads per warp from an L1-resident 64 KiB buffer;
// the pattern (lane -> 16-byte slot) is fixed per kernel.
#include <cuda_runtime.h>
#include <stdio.h>

constexpr int ITERS = 256;
constexpr int SLOTS = 4096;   // 16-byte slots = 64 KiB (L1 resident)

// pattern ids:
//  0 consecutive 16 B per lane (512 B: 4 lines)      1 all lanes same 16 B
//  2 8 lanes per line, 4 lines, lanes interleaved (lane%4 -> line)
//  3 lanes 0-7 line 0, 8-15 line 1, ... (grouped)    4 every lane its own line
//  5 two lanes per line, 16 lines                     6 13 active lanes, own lines
//  7 13 active lanes, 4 lines                         8 same as 0 but 128-bit nc allocate
__device__ __forceinline__ int slot_of(int pat, int lane) {
  switch (pat) {
    case 0: return lane;
    case 1: return 0;
    case 2: return (lane & 3) * 8 + (lane >> 2);
    case 3: return lane;                      // identical to 0 (lanes 8k..8k+7 -> line k)
    case 4: return lane * 8;
    case 5: return (lane >> 1) * 8 + (lane & 1);
    case 6: return lane * 8;
    case 7: return (lane & 3) * 8 + ((lane >> 2) & 7);
    default: return lane;
  }
}

template <int PAT, bool V8>
__global__ void load_kernel(const float4* __restrict__ buf, float* out) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const bool active = (PAT == 6 || PAT == 7) ? lane < 13 : true;
  float acc = 0.f;
  int base = (warp * 37) % (SLOTS / 64) * 64;
  for (int it = 0; it < ITERS; ++it) {
    const int s = (base + slot_of(PAT, lane) * (V8 ? 2 : 1)) % SLOTS;
    if (active) {
      if (V8) {
        float a0, a1, a2, a3, a4, a5, a6, a7;
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6),
                       "=f"(a7) : "l"(buf + s));
        acc += a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
      } else {
        float a0, a1, a2, a3;
        asm volatile("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3) : "l"(buf + s));
        acc += a0 + a1 + a2 + a3;
      }
    }
    base = (base + 64) % SLOTS;
  }
  if (acc == 1234.5f) out[0] = acc;
}

template <int PAT, bool V8>
void run(const float4* buf, float* out, const char* name) {
  load_kernel<PAT, V8><<<148, 256>>>(buf, out);
  cudaDeviceSynchronize();
  printf("%s\n", name);
}

int main() {
  float4* buf;
  float* out;
  cudaMalloc(&buf, 2 * SLOTS * sizeof(float4));
  cudaMemset(buf, 0, 2 * SLOTS * sizeof(float4));
  cudaMalloc(&out, 4);
  run<0, false>(buf, out, "p0 v4 consecutive");
  run<1, false>(buf, out, "p1 v4 same");
  run<2, false>(buf, out, "p2 v4 4 lines interleaved");
  run<4, false>(buf, out, "p4 v4 32 lines");
  run<5, false>(buf, out, "p5 v4 16 lines x2");
  run<6, false>(buf, out, "p6 v4 13 lanes own lines");
  run<7, false>(buf, out, "p7 v4 13 lanes 4 lines");
  run<0, true>(buf, out, "p0 v8 consecutive");
  run<4, true>(buf, out, "p4 v8 32 lines");
  run<6, true>(buf, out, "p6 v8 13 lanes own lines");
  return 0;
}
