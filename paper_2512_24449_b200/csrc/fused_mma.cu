// fused_mma.cu — tensor-core fused decompress + GEMV for the default format
// (pack size 16, head_dim 128, 64-token blocks).
//
// Pipeline (per CTA = 4 warps, one (sequence, kv-head) unit, a contiguous
// range of its blocks):
//   * a ring of S shared-memory slots is filled by 1-D TMA bulk copies
//     (cp.async.bulk + mbarrier complete_tx) issued by one elected thread —
//     S-1 blocks are in flight while one is decoded;
//   * warp r owns row-group r (16 tokens) of the current block: it prefix-scans
//     the 4-bit widths into a per-warp (bit offset, width,
//     1024-min) descriptor table, then walks the row-group in 16 tiles of
//     8 packs (8 channels x 16 tokens);
//   * each lane decodes 4 consecutive tokens of one pack straight into an
//     m16n8k16 fragment: two aligned smem words + funnel shift give the 4w-bit
//     window, PRMT/LOP3 place the fields under the fp16 magic exponent
//     (0x6400 = 1024) and one HSUB2 with (1024 - min) leaves the exact integer
//     code (codes < 2048 are exact in fp16);
//   * V: out[g][c] += sum_t (w_t*s_t)[g] * code[t][c] is an MMA with
//     A = w*s split into fp16 hi+lo rows (16 rows = 8 query heads x {hi, lo}),
//     B = codes (k = tokens, the pack direction), fp32 accumulators in registers
//     across all blocks of the CTA; sum_t w_t*z_t is a separate per-head scalar;
//   * K: the reduction runs over channels, across packs.  A first
//     MMA with a 0/1 permutation matrix transposes the decoded tile (its fp16
//     C/D fragment is exactly the A fragment of the next MMA), a second MMA
//     multiplies by q split into fp16 hi+lo columns (GQA: 4 query heads per
//     n8 tile).  score = s_t * acc + z_t * sum(q).
// Blocks whose packs are wider than 5 bits or whose codes exceed 2047 take a
// scalar path inside the same launch (never with the default rel 0.1 / 0.2).
#include "pkv_common.cuh"

using namespace pkv;

namespace {

constexpr int kRows = 64, kD = 128, kP = 16;
constexpr int kNib = 8, kMin = 8 + 256, kPar = kMin + 1024, kHdr = kPar + 256;  // 1544
constexpr int kMaxB = kHdr + 512 * 30;                                          // 16904
constexpr int kSlot = ((kMaxB + 15) / 16) * 16 + 16;                            // 16928
constexpr int kWarps = 4;
constexpr int kStages = 4;
constexpr int kBpc = 16;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// D(f16x2 x2) = A(16x16 f16) * B(16x8 f16) + 0
__device__ __forceinline__ void mma_f16(uint32_t (&d)[2], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%8,%9};\n"
      : "=r"(d[0]), "=r"(d[1])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(0u), "r"(0u));
}
// C(f32 x4) += A(16x16 f16) * B(16x8 f16)
__device__ __forceinline__ void mma_f32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
  return uint32_t(__half_as_ushort(lo)) | (uint32_t(__half_as_ushort(hi)) << 16);
}
__device__ __forceinline__ void split_hilo(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}
__device__ __forceinline__ uint32_t hsub2_u32(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ float h2f(uint32_t bits16) { return __half2float(__ushort_as_half(uint16_t(bits16))); }

// Decode 4 consecutive w-bit fields (tokens 4tq..4tq+3 of one pack) at bit b0
// of the slot into two f16x2 fragment registers holding the exact codes:
// r01 = (code0, code1), r23 = (code2, code3).  Valid for w <= 5.
__device__ __forceinline__ void decode4(const uint32_t* __restrict__ words, uint32_t b0, uint32_t w,
                                        uint32_t cm2, uint32_t& r01, uint32_t& r23) {
  const uint32_t i = b0 >> 5;
  const uint32_t x = __funnelshift_r(words[i], words[i + 1], b0);
  const uint32_t m = (1u << w) - 1u;
  const uint32_t MM = m | (m << 16);
  const uint32_t t = x << (16u - w);
  const uint32_t y = __byte_perm(x, t, 0x7610);
  const uint32_t h01 = (y & MM) | 0x64006400u;
  const uint32_t h23 = ((y >> (2u * w)) & MM) | 0x64006400u;
  r01 = hsub2_u32(h01, cm2);
  r23 = hsub2_u32(h23, cm2);
}

// Generic scalar read of field `t` of a pack (any width <= 15).
__device__ __forceinline__ uint32_t field(const uint32_t* __restrict__ words, uint32_t bitpos, uint32_t w,
                                          uint32_t t) {
  const uint32_t b = bitpos + t * w;
  const uint32_t i = b >> 5;
  const uint32_t x = __funnelshift_r(words[i], words[i + 1], b);
  return x & ((1u << w) - 1u);
}

struct RowDesc {
  bool fast;
};

// Per-warp header parse of row-group rg: writes dc[pos] = {bitpos | w << 24,
// half2(1024 - min)} for the 128 physical packs of the row-group and
// mn[pos] = min.  Returns whether the whole row-group fits the fast path.
__device__ __forceinline__ bool parse_rowgroup(const uint8_t* __restrict__ blk, int rg, int lane,
                                               uint2* __restrict__ dc, uint16_t* __restrict__ mn) {
  // widths of all 4 row-groups: lane owns nibble bytes 2l, 2l+1 of each
  uint32_t nb[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) nb[r] = *(const uint16_t*)(blk + kNib + 64 * r + 2 * lane);
  // SWAR sum of 4 nibbles for row-groups (0,1) and (2,3)
  uint32_t v01 = nb[0] | (nb[1] << 16), v23 = nb[2] | (nb[3] << 16);
  v01 = (v01 & 0x0f0f0f0fu) + ((v01 >> 4) & 0x0f0f0f0fu);
  v23 = (v23 & 0x0f0f0f0fu) + ((v23 >> 4) & 0x0f0f0f0fu);
  v01 = (v01 & 0x00ff00ffu) + ((v01 >> 8) & 0x00ff00ffu);
  v23 = (v23 & 0x00ff00ffu) + ((v23 >> 8) & 0x00ff00ffu);
  uint32_t s01 = v01, s23 = v23;  // per-lane, packed 16-bit sums
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s01 += __shfl_xor_sync(PKV_FULL, s01, o);
    s23 += __shfl_xor_sync(PKV_FULL, s23, o);
  }
  const uint32_t tot[4] = {s01 & 0xffff, s01 >> 16, s23 & 0xffff, s23 >> 16};
  uint32_t base = kHdr;
#pragma unroll
  for (int r = 0; r < 4; ++r)
    if (r < rg) base += 2 * tot[r];  // payload bytes = k*w/8 = 2w at k = 16
  // own row-group: lane's 4 consecutive packs 4l..4l+3
  const uint32_t nbo = nb[rg];
  const uint32_t w0 = nbo & 15, w1 = (nbo >> 4) & 15, w2 = (nbo >> 8) & 15, w3 = (nbo >> 12) & 15;
  const uint32_t lsum = 2 * (w0 + w1 + w2 + w3);
  uint32_t inc = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(PKV_FULL, inc, o);
    if (lane >= o) inc += y;
  }
  uint32_t off = base + inc - lsum;  // byte offset (from slot start) of pack 4l
  const uint2 mins = *(const uint2*)(blk + kMin + 256 * rg + 8 * lane);
  const uint32_t mnv[4] = {mins.x & 0xffff, mins.x >> 16, mins.y & 0xffff, mins.y >> 16};
  const uint32_t wv[4] = {w0, w1, w2, w3};
  bool ok = true;
  uint2 d[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ok &= (wv[i] <= 5u) && (mnv[i] + (1u << wv[i]) - 1u <= 2047u);
    const __half c = __int2half_rn(1024 - int(mnv[i]));
    d[i].x = (off * 8u) | (wv[i] << 24);
    d[i].y = pack_h2(c, c);
    off += 2 * wv[i];
  }
  uint4* dc4 = (uint4*)(dc + 4 * lane);
  dc4[0] = make_uint4(d[0].x, d[0].y, d[1].x, d[1].y);
  dc4[1] = make_uint4(d[2].x, d[2].y, d[3].x, d[3].y);
  *(uint2*)(mn + 4 * lane) = mins;
  __syncwarp();
  return __all_sync(PKV_FULL, ok);
}

struct Ring {
  uint64_t* full;
  uint64_t* empty;
  uint8_t* slots;
};

__device__ __forceinline__ void issue_block(const Ring& R, int i, const pkv_layer_t& L, int64_t tab, int j) {
  const int s = i % kStages;
  const int64_t off = L.blk_off[tab + j];
  const uint32_t bytes = uint32_t((L.blk_len[tab + j] + 15) & ~15);
  mbar_expect_tx(&R.full[s], bytes);
  tma_load_1d(R.slots + size_t(s) * kSlot, L.arena + off, bytes, &R.full[s]);
}

// Shared ring setup + producer schedule; calls body(i, j, slot) for each block.
template <class Body>
__device__ __forceinline__ void run_blocks(const Ring& R, const pkv_layer_t& L, int64_t tab, int j0, int nb,
                                           Body&& body) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0)
    for (int i = 0; i < kStages - 1 && i < nb; ++i) issue_block(R, i, L, tab, j0 + i);
  for (int i = 0; i < nb; ++i) {
    if (threadIdx.x == 0 && i + kStages - 1 < nb) {
      if (i >= 1) mbar_wait(&R.empty[(i - 1) % kStages], uint32_t(((i - 1) / kStages) & 1));
      issue_block(R, i + kStages - 1, L, tab, j0 + i + kStages - 1);
    }
    const int s = i % kStages;
    mbar_wait(&R.full[s], uint32_t((i / kStages) & 1));
    body(i, j0 + i, R.slots + size_t(s) * kSlot);
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.empty[s]);
  }
  (void)warp;
}

__device__ __forceinline__ uint8_t* setup_ring(uint8_t* smem, Ring& R) {
  R.slots = smem;
  R.full = (uint64_t*)(smem + size_t(kStages) * kSlot);
  R.empty = R.full + kStages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], kWarps);
    }
    fence_barrier_init();
  }
  return (uint8_t*)(R.empty + kStages);
}

constexpr size_t kRingBytes = size_t(kStages) * kSlot + 2 * kStages * 8;
constexpr size_t kWarpDesc = 128 * 8 + 128 * 2;  // dc + mn per warp

// ======================================================================= V
template <int GN>  // GN = max query heads per kv head handled (<= 8)
__global__ void __launch_bounds__(kWarps * 32) fused_v_mma_kernel(pkv_layer_t L, const float* __restrict__ w,
                                                                   int G, int64_t wstride,
                                                                   float* __restrict__ part, int bpc,
                                                                   int nsplit) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  uint8_t* rest = setup_ring(smem, R);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  uint2* dc = (uint2*)(rest + warp * kWarpDesc);
  uint16_t* mn = (uint16_t*)(rest + warp * kWarpDesc + 128 * 8);
  __syncthreads();

  const int u = blockIdx.y, b = u / L.heads, h = u % L.heads, U = L.batch * L.heads;
  const int Hq = L.heads * G;
  const int nbk = L.nblk[b];
  const int j0 = blockIdx.x * bpc, j1 = min(nbk, j0 + bpc);
  const int64_t tab = (int64_t(1) * U + u) * L.max_blocks;
  const int rg = warp;
  const bool head_ok = gi < G;
  const float* wrow = w + (int64_t(b) * Hq + int64_t(h) * G + (head_ok ? gi : 0)) * wstride;

  float acc[16][4];
#pragma unroll
  for (int t = 0; t < 16; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
  float zacc = 0.f;

  run_blocks(R, L, tab, j0, max(0, j1 - j0), [&](int i, int j, const uint8_t* blk) {
    // weights of this lane's 4 tokens (hot in L2; issued before the header parse)
    const int tok0 = rg * 16 + 4 * tq;
    float4 wv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (head_ok) wv = *(const float4*)(wrow + int64_t(j) * kRows + tok0);
    const bool fast = parse_rowgroup(blk, rg, lane, dc, mn);
    // per-token params (scale, zp) of tokens tok0..tok0+3
    const uint2 p01 = *(const uint2*)(blk + kPar + 4 * tok0);
    const uint2 p23 = *(const uint2*)(blk + kPar + 4 * tok0 + 8);
    const float s0 = h2f(p01.x & 0xffff), z0 = h2f(p01.x >> 16), s1 = h2f(p01.y & 0xffff), z1 = h2f(p01.y >> 16);
    const float s2 = h2f(p23.x & 0xffff), z2 = h2f(p23.x >> 16), s3 = h2f(p23.y & 0xffff), z3 = h2f(p23.y >> 16);
    zacc = fmaf(wv.x, z0, fmaf(wv.y, z1, fmaf(wv.z, z2, fmaf(wv.w, z3, zacc))));
    const float ws0 = wv.x * s0, ws1 = wv.y * s1, ws2 = wv.z * s2, ws3 = wv.w * s3;
    const uint32_t* words = (const uint32_t*)blk;
    if (fast) {
      __half h0, l0, h1, l1, h2_, l2, h3, l3;
      split_hilo(ws0, h0, l0);
      split_hilo(ws1, h1, l1);
      split_hilo(ws2, h2_, l2);
      split_hilo(ws3, h3, l3);
      // A rows: gi = hi part of head gi, gi+8 = lo part; k = (4tq,4tq+1 | 4tq+2,4tq+3)
      const uint32_t a[4] = {pack_h2(h0, h1), pack_h2(l0, l1), pack_h2(h2_, h3), pack_h2(l2, l3)};
#pragma unroll
      for (int t = 0; t < 16; ++t) {
        const uint2 d = dc[8 * t + gi];
        const uint32_t wd = d.x >> 24;
        uint32_t b0, b1;
        decode4(words, (d.x & 0xffffffu) + 4u * tq * wd, wd, d.y, b0, b1);
        mma_f32(acc[t], a, b0, b1);
      }
    } else {
      // scalar path: this lane owns head gi, channels 8t+2tq, 8t+2tq+1 (hi row)
      float wsr[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const int tok = rg * 16 + r;
        const uint32_t pr = *(const uint32_t*)(blk + kPar + 4 * tok);
        wsr[r] = head_ok ? wrow[int64_t(j) * kRows + tok] * h2f(pr & 0xffff) : 0.f;
      }
#pragma unroll
      for (int t = 0; t < 16; ++t) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int pos = 8 * t + 2 * tq + e;
          const uint2 d = dc[pos];
          const uint32_t wd = d.x >> 24, bp = d.x & 0xffffffu, m0 = mn[pos];
          float a = 0.f;
          for (int r = 0; r < 16; ++r) a = fmaf(wsr[r], float(m0 + field(words, bp, wd, r)), a);
          acc[t][e] += a;
        }
      }
    }
    (void)i;
  });

  // ---- fixed-order cross-warp reduction (after the ring drained)
  __syncthreads();
  float* red = (float*)smem;  // [kWarps][GN][kD]
  float* zred = red + kWarps * GN * kD;  // [kWarps][GN]
  zacc += __shfl_xor_sync(PKV_FULL, zacc, 1);
  zacc += __shfl_xor_sync(PKV_FULL, zacc, 2);
  if (head_ok) {
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int c = 8 * t + 2 * tq;
      red[(warp * GN + gi) * kD + c] = acc[t][0] + acc[t][2];
      red[(warp * GN + gi) * kD + c + 1] = acc[t][1] + acc[t][3];
    }
    if (tq == 0) zred[warp * GN + gi] = zacc;
  }
  __syncthreads();
  const int nr = (blockIdx.x == 0) ? L.nres[b] : 0;
  const uint16_t* vr = L.stage + (int64_t(1) * U + u) * L.buffer * kD;
  for (int e = threadIdx.x; e < G * (kD + 1); e += blockDim.x) {
    const int g = e / (kD + 1), c = e % (kD + 1);
    float s = 0.f;
    if (c < kD) {
#pragma unroll
      for (int wv = 0; wv < kWarps; ++wv) s += red[(wv * GN + g) * kD + c];
      const float* wr = w + (int64_t(b) * Hq + int64_t(h) * G + g) * wstride + int64_t(nbk) * kRows;
      for (int t = 0; t < nr; ++t) s = fmaf(wr[t], __half2float(__ushort_as_half(vr[t * kD + c])), s);
    } else {
#pragma unroll
      for (int wv = 0; wv < kWarps; ++wv) s += zred[wv * GN + g];
    }
    part[((int64_t(u) * nsplit + blockIdx.x) * G + g) * (kD + 1) + c] = s;
  }
}

__global__ void fused_v_mma_finalize(const float* __restrict__ part, int U, int G, int nsplit,
                                     float* __restrict__ out) {
  const int64_t total = int64_t(U) * G * kD;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(e % kD);
    const int64_t ug = e / kD;
    const int gq = int(ug % G);
    const int64_t u = ug / G;
    float s = 0.f, z = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float* pp = part + ((u * nsplit + sp) * G + gq) * (kD + 1);
      s += pp[c];
      z += pp[kD];
    }
    out[e] = s + z;
  }
}

// ======================================================================= K
template <int NT>  // n8 tiles of (head, hi/lo) columns: 1 for G <= 4, 2 for G <= 8
__global__ void __launch_bounds__(kWarps * 32) fused_k_mma_kernel(pkv_layer_t L, const float* __restrict__ q,
                                                                   int G, float* __restrict__ scores,
                                                                   int64_t sstride, int bpc) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  uint8_t* rest = setup_ring(smem, R);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  uint2* dc = (uint2*)(rest + warp * kWarpDesc);
  uint16_t* mn = (uint16_t*)(rest + warp * kWarpDesc + 128 * 8);
  float* sq = (float*)(rest + kWarps * kWarpDesc);  // [G][kD]
  float* sqsum = sq + 8 * kD;                        // [G]

  const int u = blockIdx.y, b = u / L.heads, h = u % L.heads, U = L.batch * L.heads;
  const int Hq = L.heads * G;
  const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * kD;
  for (int e = threadIdx.x; e < G * kD; e += blockDim.x) sq[e] = qu[e];
  __syncthreads();
  for (int g = warp; g < G; g += kWarps) {
    float s = 0.f;
    for (int c = lane; c < kD; c += 32) s += sq[g * kD + c];
    s = warp_sum(s);
    if (lane == 0) sqsum[g] = s;
  }
  // B2 fragments: k-step s covers K-layout physical positions 16s..16s+15;
  // column n = gi -> head (nt*4 + gi/2), part hi (gi even) / lo (gi odd).
  uint32_t bq[NT][8][2];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int g = nt * 4 + (gi >> 1);
    const bool lo = gi & 1;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        __half v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int pos = 16 * s + 2 * tq + 8 * r + e;
          const int c = kpos_to_col(pos, kD);
          const float x = g < G ? sq[g * kD + c] : 0.f;
          __half hh, ll;
          split_hilo(x, hh, ll);
          v[e] = lo ? ll : hh;
        }
        bq[nt][s][r] = pack_h2(v[0], v[1]);
      }
    }
  }
  // A1: permutation matrix, row r <- k-index kappa with pi(2tq)=4tq, pi(2tq+1)=4tq+1,
  // pi(2tq+8)=4tq+2, pi(2tq+9)=4tq+3  (rows = tokens of the row-group)
  uint32_t aperm[4];
  {
    const uint16_t one = 0x3c00;
    auto e = [&](int row, int kk) -> uint16_t {
      const int t4 = kk & 7;  // kk in {2tq', 2tq'+1} or {2tq'+8, 2tq'+9}
      const int tqq = t4 >> 1, lo = t4 & 1, hi8 = kk >= 8;
      const int tok = 4 * tqq + 2 * hi8 + lo;
      return tok == row ? one : 0;
    };
    const int c0 = 2 * tq;
    aperm[0] = uint32_t(e(gi, c0)) | (uint32_t(e(gi, c0 + 1)) << 16);
    aperm[1] = uint32_t(e(gi + 8, c0)) | (uint32_t(e(gi + 8, c0 + 1)) << 16);
    aperm[2] = uint32_t(e(gi, c0 + 8)) | (uint32_t(e(gi, c0 + 9)) << 16);
    aperm[3] = uint32_t(e(gi + 8, c0 + 8)) | (uint32_t(e(gi + 8, c0 + 9)) << 16);
  }
  __syncthreads();

  const int nbk = L.nblk[b];
  const int j0 = blockIdx.x * bpc, j1 = min(nbk, j0 + bpc);
  const int64_t tab = (int64_t(0) * U + u) * L.max_blocks;
  const int rg = warp;
  float* srow = scores + (int64_t(b) * Hq + int64_t(h) * G) * sstride;

  run_blocks(R, L, tab, j0, max(0, j1 - j0), [&](int i, int j, const uint8_t* blk) {
    const bool fast = parse_rowgroup(blk, rg, lane, dc, mn);
    const uint32_t* words = (const uint32_t*)blk;
    const int tA = rg * 16 + gi, tB = tA + 8;
    const uint32_t pA = *(const uint32_t*)(blk + kPar + 4 * tA);
    const uint32_t pB = *(const uint32_t*)(blk + kPar + 4 * tB);
    const float sA = h2f(pA & 0xffff), zA = h2f(pA >> 16), sB = h2f(pB & 0xffff), zB = h2f(pB >> 16);
    if (fast) {
      float acc[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.f;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        uint32_t dt[2][2];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const uint2 d = dc[16 * s + 8 * half + gi];
          const uint32_t wd = d.x >> 24;
          uint32_t b0, b1;
          decode4(words, (d.x & 0xffffffu) + 4u * tq * wd, wd, d.y, b0, b1);
          mma_f16(dt[half], aperm, b0, b1);  // transpose: rows = tokens, cols = 8 packs
        }
        const uint32_t a2[4] = {dt[0][0], dt[0][1], dt[1][0], dt[1][1]};
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mma_f32(acc[nt], a2, bq[nt][s][0], bq[nt][s][1]);
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int g = nt * 4 + tq;
        if (g < G) {
          srow[int64_t(g) * sstride + int64_t(j) * kRows + tA] = fmaf(sA, acc[nt][0] + acc[nt][1], zA * sqsum[g]);
          srow[int64_t(g) * sstride + int64_t(j) * kRows + tB] = fmaf(sB, acc[nt][2] + acc[nt][3], zB * sqsum[g]);
        }
      }
    } else {
      // scalar path: this lane computes tokens tA, tB for heads tq (+4)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int g = nt * 4 + tq;
        if (g >= G) continue;
        float aA = 0.f, aB = 0.f;
        for (int pos = 0; pos < 128; ++pos) {
          const uint2 d = dc[pos];
          const uint32_t wd = d.x >> 24, bp = d.x & 0xffffffu, m0 = mn[pos];
          const float qv = sq[g * kD + kpos_to_col(pos, kD)];
          aA = fmaf(float(m0 + field(words, bp, wd, gi)), qv, aA);
          aB = fmaf(float(m0 + field(words, bp, wd, gi + 8)), qv, aB);
        }
        srow[int64_t(g) * sstride + int64_t(j) * kRows + tA] = fmaf(sA, aA, zA * sqsum[g]);
        srow[int64_t(g) * sstride + int64_t(j) * kRows + tB] = fmaf(sB, aB, zB * sqsum[g]);
      }
    }
    (void)i;
  });

  if (blockIdx.x == 0) {  // uncompressed residue, same launch
    const int nr = L.nres[b];
    const uint16_t* kr = L.stage + (int64_t(0) * U + u) * L.buffer * kD;
    for (int t = warp; t < nr; t += kWarps) {
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
        for (int c = lane; c < kD; c += 32) a = fmaf(__half2float(__ushort_as_half(kr[t * kD + c])), sq[g * kD + c], a);
        a = warp_sum(a);
        if (lane == 0) srow[int64_t(g) * sstride + int64_t(nbk) * kRows + t] = a;
      }
    }
  }
}

constexpr size_t k_smem_bytes() { return kRingBytes + kWarps * kWarpDesc + (8 * kD + 8) * 4; }
template <int GN>
constexpr size_t v_smem_bytes() {
  const size_t ring = kRingBytes + kWarps * kWarpDesc;
  const size_t red = size_t(kWarps) * GN * kD * 4 + kWarps * GN * 4;
  return ring > red ? ring : red;
}

}  // namespace

// Entry points used by fused.cu for the default format (k = 16, D = 128, G <= 8).
bool pkv_mma_supported(const pkv_layer_t* L, int G, int64_t stride) {
  return L->pack_size == kP && L->head_dim == kD && L->block == kRows && G >= 1 && G <= 8 && stride % 4 == 0;
}

int pkv_mma_fused_k(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
                    cudaStream_t s) {
  const size_t smem = k_smem_bytes();
  dim3 grid(max(1, (nblocks + kBpc - 1) / kBpc), L->batch * L->heads);
  if (G <= 4) {
    cudaFuncSetAttribute(fused_k_mma_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    fused_k_mma_kernel<1><<<grid, kWarps * 32, smem, s>>>(*L, q, G, scores, sstride, kBpc);
  } else {
    cudaFuncSetAttribute(fused_k_mma_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    fused_k_mma_kernel<2><<<grid, kWarps * 32, smem, s>>>(*L, q, G, scores, sstride, kBpc);
  }
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_k_scores(mma)");
}

int64_t pkv_mma_v_scratch(const pkv_layer_t* L, int nblocks, int G) {
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  return int64_t(L->batch) * L->heads * nsplit * G * (kD + 1) * 4;
}

int pkv_mma_fused_v(const pkv_layer_t* L, int nblocks, const float* w, int G, int64_t wstride, float* out,
                    float* part, cudaStream_t s) {
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  dim3 grid(nsplit, L->batch * L->heads);
  const size_t smem = v_smem_bytes<8>();
  cudaFuncSetAttribute(fused_v_mma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  fused_v_mma_kernel<8><<<grid, kWarps * 32, smem, s>>>(*L, w, G, wstride, part, kBpc, nsplit);
  const int64_t total = int64_t(L->batch) * L->heads * G * kD;
  const int fgrid = int((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  fused_v_mma_finalize<<<fgrid, 256, 0, s>>>(part, L->batch * L->heads, G, nsplit, out);
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_v_output(mma)");
}
