// Probe: throughput of a 1-D TMA bulk-copy ring (one producer lane, C consumer
// warps that only wait + release), as a function of CTAs/SM, ring slots and
// copy size.  Prints GB/s.
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void feed(const uint8_t* src, int64_t nblk_total, int bytes, int slots, int stride_blocks, int nconsumer,
                     unsigned long long* sink, int nprod) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 64;
  uint8_t* ring = sm + 1024;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int64_t per = nblk_total / gridDim.x;
  const int64_t b0 = per * blockIdx.x;
  if (warp >= nconsumer) {
    const int pw = warp - nconsumer;
    if (lane == 0) {
      for (int64_t t = pw; t < per; t += nprod) {
        const int s = int(t % slots);
        if (t >= slots) {
          const uint32_t par = uint32_t(((t / slots) - 1) & 1);
          asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(sa(&empty[s])), "r"(par) : "memory");
        }
        const int64_t gb = b0 + t;
        const int64_t blk = (gb * stride_blocks) % nblk_total;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(ring + s * bytes)),
                     "l"(src + blk * bytes), "r"(bytes), "r"(sa(&full[s])) : "memory");
      }
    }
    return;
  }
  unsigned long long acc = 0;
  for (int64_t t = warp; t < per; t += nconsumer) {
    const int s = int(t % slots);
    const uint32_t par = uint32_t((t / slots) & 1);
    asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W2;\n}\n" ::"r"(sa(&full[s])), "r"(par) : "memory");
    acc += ring[s * bytes + lane * 4];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
  }
  if (acc == 12345) sink[0] = acc;
}
int main() {
  const int64_t total_bytes = 256ll << 20;
  uint8_t* src; cudaMalloc(&src, total_bytes); cudaMemset(src, 1, total_bytes);
  unsigned long long* sink; cudaMalloc(&sink, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(feed, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int cta, slots, bytes, stride, cons, prod; };
  std::vector<Cfg> cfgs = {
    {1, 16, 4096, 1, 4, 1}, {1, 16, 4096, 1, 4, 2}, {1, 16, 4096, 1, 4, 4}, {1, 32, 4096, 1, 8, 8},
    {2, 16, 4096, 1, 4, 4}, {4, 8, 4096, 1, 4, 2}, {4, 8, 4096, 1, 4, 4}, {1, 32, 2048, 1, 4, 8}};
  for (auto c : cfgs) {
    const int64_t nblk = total_bytes / c.bytes;
    const int grid = nsm * c.cta;
    const size_t smem = 1024 + size_t(c.slots) * c.bytes;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) feed<<<grid, (c.cons + c.prod) * 32, smem>>>(src, nblk, c.bytes, c.slots, c.stride, c.cons, sink, c.prod);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int it = 0; it < reps; ++it) feed<<<grid, (c.cons + c.prod) * 32, smem>>>(src, nblk, c.bytes, c.slots, c.stride, c.cons, sink, c.prod);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes_moved = double(nblk / grid * grid) * c.bytes * reps;
    printf("cta/sm %d slots %2d bytes %6d stride %3d consumers %d producers %d : %7.1f GB/s  (%s)\n", c.cta, c.slots, c.bytes, c.stride, c.cons, c.prod,
           bytes_moved / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
