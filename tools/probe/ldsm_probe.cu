// Probe: fragment layout of ldmatrix.m16n16.x2.trans.b8 on sm_100a.
#include <cstdio>
#include <cstdint>
__global__ void probe(uint32_t* out) {
  __shared__ __align__(128) uint8_t s[32 * 16];
  for (int i = threadIdx.x; i < 512; i += 32) s[i] = uint8_t(i & 255);  // row r = i/16 (0..31), col = i%16
  __syncwarp();
  uint32_t r0, r1, r2, r3;
  uint32_t addr = (uint32_t)__cvta_generic_to_shared(s + threadIdx.x * 16);
  asm volatile("ldmatrix.sync.aligned.m16n16.x2.trans.shared.b8 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
  out[threadIdx.x * 4 + 0] = r0; out[threadIdx.x * 4 + 1] = r1;
  out[threadIdx.x * 4 + 2] = r2; out[threadIdx.x * 4 + 3] = r3;
}
int main() {
  uint32_t* d; cudaMalloc(&d, 512); probe<<<1, 32>>>(d);
  uint32_t h[128]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  for (int t = 0; t < 32; ++t) {
    printf("lane %2d:", t);
    for (int r = 0; r < 4; ++r) {
      printf("  r%d=", r);
      for (int b = 0; b < 4; ++b) { int v = (h[t*4+r] >> (8*b)) & 255; printf("(%d,%d)", v / 16, v % 16); }
    }
    printf("\n");
  }
  return 0;
}
