// mma_rate_probe.cu — legacy mma.sync tensor-core issue rates on sm_100a
// (u8 m16n8k32, u4 m16n8k64, f16 m16n8k16), to size the fused kernels'
// product stage.  Each warp runs CH independent accumulator chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate_probe mma_rate_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int KIND, int CH>
__global__ void probe(int iters, int* out, uint32_t seed) {
  int c[CH][4];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0;
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (KIND == 0)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else if (KIND == 1)
        asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.u4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0;
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 0x12345) out[0] = s;
}

template <int KIND, int CH>
void run(const char* name, int warps_per_cta, int ctas_per_sm) {
  int* d;
  cudaMalloc(&d, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<KIND, CH><<<sms * ctas_per_sm, 32 * warps_per_cta>>>(16, d, 1);
  cudaEventRecord(e0);
  probe<KIND, CH><<<sms * ctas_per_sm, 32 * warps_per_cta>>>(iters, d, 1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double n_mma = double(sms) * ctas_per_sm * warps_per_cta * iters * CH;
  const double per_sm_cycle = n_mma / sms / (ms * 1e-3 * 1.965e9);
  const int macs = KIND == 0 ? 16 * 8 * 32 : KIND == 1 ? 16 * 8 * 64 : 16 * 8 * 16;
  printf("%-10s warps/SM %3d chains %d: %.3f ms, %.3f mma/SM/cycle (@1.965GHz), %.1f TOPS\n", name,
         warps_per_cta * ctas_per_sm, CH, ms, per_sm_cycle, n_mma * macs * 2 / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  for (int w : {4, 8, 16, 32}) {
    run<0, 4>("u8k32", w, 1);
    run<1, 4>("u4k64", w, 1);
    run<2, 4>("f16k16", w, 1);
  }
  run<0, 1>("u8k32", 16, 1);
  run<0, 2>("u8k32", 16, 1);
  run<1, 1>("u4k64", 16, 1);
  return 0;
}
