// fused_i8.cu — int8 tensor-core fused decompress + GEMV for the default
// format (pack size 16, head_dim 128, 64-token blocks).
//
// CTA = 4 consumer warps + 1 producer warp, one (sequence, kv-head) unit and a
// contiguous range of its blocks.
//  * Producer (one lane): streams the unit's PackedBlocks with 1-D TMA bulk
//    copies (cp.async.bulk + mbarrier complete_tx) into a 64 KB byte ring.
//    Blocks are packed back to back (16-byte aligned), so ~15 typical 4 KB
//    blocks are in flight per CTA.
//  * Consumer warp w owns blocks w, w+4, ...: it prefix-scans the 512 4-bit
//    pack widths into a per-warp descriptor table
//    (payload bit position | width | minimum), then decodes.
//  * Each lane decodes 8 consecutive tokens of one pack per step: two
//    aligned smem words + funnel shift give the 8w-bit window, and two
//    PRMT/shift rounds place 4 fields per register into byte lanes; adding
//    min*0x01010101 gives the exact uint8 codes.
//  * The codes feed mma.sync.m16n8k32 (IMMA, u8 x {u8,s8} -> s32).  The other
//    operand is an exact fixed-point integer: the query (K) or w*scale (V)
//    scaled by a per-CTA power of two and split into 3 byte digits (two
//    unsigned low bytes and a signed top byte), so every accumulation is
//    exact in int32 and the only rounding is the 23-bit fixed point.
//  * V: D[channels][digit,head] += codes[channels][tokens] x
//    digits[tokens][digit,head]; tokens are the k dimension (the pack
//    direction), 32 tokens = 2 row-groups per MMA.
//  * K: the reduction runs over channels.  An IMMA with a 0/1
//    permutation matrix transposes each 16-token x 16-channel tile of codes
//    (its s32 C fragment holds token rows x channel pairs), three IMADs pack
//    them into the next IMMA's A fragment, and that IMMA multiplies by the
//    query digits.  score = s_t * (acc / 2^S) + z_t * sum(q).
// Blocks with a pack wider than 4 bits or a code above 255 take a scalar
// path inside the same launch (never at the default rel 0.1 / 0.2).
#include "pkv_common.cuh"

using namespace pkv;

namespace {

constexpr int kRows = 64, kD = 128, kP = 16;
constexpr int kNib = 8, kMin = 8 + 256, kPar = kMin + 1024, kHdr = kPar + 256;  // 1544
constexpr int kRing = 48 * 1024;
constexpr int kTickets = 16;
constexpr int kCW = 4;
constexpr int kThreads = (kCW + 1) * 32;
constexpr int kBpc = 32;

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
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kCW * 32) : "memory");
}

// D = A(u8 16x32) * B(u8 32x8) + C
__device__ __forceinline__ void imma_uu(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// D = A(u8) * B(s8) + C
__device__ __forceinline__ void imma_us(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// D = A(u8) * B(u8), C = 0
__device__ __forceinline__ void imma_uu0(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};\n"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "r"(0));
}

__device__ __forceinline__ float h2f(uint32_t bits16) { return __half2float(__ushort_as_half(uint16_t(bits16))); }

// byte `p` (runtime 0..3) of each of x0..x3 packed into one register
__device__ __forceinline__ uint32_t gather_byte(uint32_t x0, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t sel) {
  const uint32_t t01 = __byte_perm(x0, x1, sel);
  const uint32_t t23 = __byte_perm(x2, x3, sel);
  return __byte_perm(t01, t23, 0x5410);
}

// ---------------------------------------------------------------- block parse
// Whole-block parse by one warp: lane l owns the 16 consecutive physical packs
// 16l..16l+15.  desc[p] = payload bit position (from the block start, 18 bits)
// | width << 18 | min << 22.  Returns true when every pack fits the fast path
// (width <= 4 and min + 2^w - 1 <= 255).
__device__ __forceinline__ bool parse_block(const uint8_t* __restrict__ blk, int lane, uint32_t* __restrict__ desc) {
  const uint2 nb = *(const uint2*)(blk + kNib + 8 * lane);
  // payload bytes of the lane's 16 packs = 2 * sum(widths)  (k = 16)
  uint32_t a = (nb.x & 0x0f0f0f0fu) + ((nb.x >> 4) & 0x0f0f0f0fu);
  uint32_t b = (nb.y & 0x0f0f0f0fu) + ((nb.y >> 4) & 0x0f0f0f0fu);
  a += b;
  a = (a & 0x00ff00ffu) + ((a >> 8) & 0x00ff00ffu);
  const uint32_t lsum = 2u * ((a & 0xffffu) + (a >> 16));
  uint32_t inc = lsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(PKV_FULL, inc, o);
    if (lane >= o) inc += y;
  }
  uint32_t off = kHdr + inc - lsum;
  const uint2* mp = (const uint2*)(blk + kMin + 32 * lane);
  uint32_t mins[8];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint2 v = mp[q];
    mins[2 * q] = v.x;
    mins[2 * q + 1] = v.y;
  }
  bool ok = true;
  uint32_t d[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t w = ((i < 8 ? nb.x : nb.y) >> (4 * (i & 7))) & 15u;
    const uint32_t mn = (mins[i >> 1] >> (16 * (i & 1))) & 0xffffu;
    ok &= (w <= 4u) && (mn + (1u << w) - 1u <= 255u);
    d[i] = (off * 8u) | (w << 18) | (mn << 22);
    off += 2u * w;
  }
  uint4* d4 = (uint4*)(desc + 16 * lane);
#pragma unroll
  for (int q = 0; q < 4; ++q) d4[q] = make_uint4(d[4 * q], d[4 * q + 1], d[4 * q + 2], d[4 * q + 3]);
  __syncwarp();
  return __all_sync(PKV_FULL, ok);
}

// Four fields at stride w (w <= 4) in the low bits of x -> one byte each,
// plus the pack minimum: exact uint8 codes (byte e = field e).
__device__ __forceinline__ uint32_t spread4(uint32_t x, uint32_t s1, uint32_t s2, uint32_t m4, uint32_t mr) {
  const uint32_t y = __byte_perm(x, x << s1, 0x7610);  // fields 0,1 low half; 2,3 high half
  const uint32_t z = __byte_perm(y, y << s2, 0x7250);  // one field per byte
  return (z & m4) + mr;
}

// All 16 fields of the pack described by `d` (w <= 4) as uint8 codes:
// r[q] holds tokens 4q..4q+3 (byte e = token 4q+e).
__device__ __forceinline__ void decode16(const uint32_t* __restrict__ words, uint32_t d, uint32_t (&r)[4]) {
  const uint32_t bo = d & 0x3ffffu;
  const uint32_t w = (d >> 18) & 15u;
  const uint32_t* p = words + (bo >> 5);
  const uint32_t w0 = p[0], w1 = p[1], w2 = p[2];
  const uint32_t xlo = __funnelshift_r(w0, w1, bo);
  const uint32_t xmid = __funnelshift_r(w1, w2, bo);
  const uint32_t xhi = __funnelshift_rc(xlo, xmid, 8u * w);  // fields 8..15 (clamped at 32 for w = 4)
  const uint32_t m4 = (0x01010101u << w) - 0x01010101u;
  const uint32_t mr = (d >> 22) * 0x01010101u;
  const uint32_t s2 = 8u - w, s1 = 2u * s2, s3 = 4u * w;
  r[0] = spread4(xlo, s1, s2, m4, mr);
  r[1] = spread4(xlo >> s3, s1, s2, m4, mr);
  r[2] = spread4(xhi, s1, s2, m4, mr);
  r[3] = spread4(xhi >> s3, s1, s2, m4, mr);
}

// Generic scalar field read (any width <= 15) from a block at any alignment.
__device__ __forceinline__ uint32_t field_bytes(const uint8_t* __restrict__ blk, uint32_t bitpos, uint32_t w) {
  if (w == 0) return 0;
  const uint8_t* p = blk + (bitpos >> 3);
  const uint32_t sh = bitpos & 7;
  const uint32_t v = uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16);
  return (v >> sh) & ((1u << w) - 1u);
}
__device__ __forceinline__ uint32_t pack_min(const uint8_t* __restrict__ blk, int p) {
  return uint32_t(blk[kMin + 2 * p]) | (uint32_t(blk[kMin + 2 * p + 1]) << 8);
}

// ---------------------------------------------------------------- ring
struct Ring {
  uint8_t* data;
  uint64_t* full;
  uint64_t* empty;
  uint32_t* start;  // [kTickets] ring offset of each ticket's block
  uint32_t* abs;    // [kTickets] producer-private absolute start
};

__device__ __forceinline__ uint8_t* setup_ring(uint8_t* smem, Ring& R) {
  R.data = smem;
  R.full = (uint64_t*)(smem + kRing);
  R.empty = R.full + kTickets;
  R.start = (uint32_t*)(R.empty + kTickets);
  R.abs = R.start + kTickets;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTickets; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], 1);
    }
    fence_barrier_init();
  }
  return (uint8_t*)(R.abs + kTickets);
}
constexpr size_t kRingBytes = kRing + kTickets * 8 * 2 + kTickets * 4 * 2;

// Single-lane producer: block i -> ticket i % kTickets, placed back to back in
// the byte ring; waits (in ticket order) for releases when out of tickets or bytes.
__device__ void produce(const Ring& R, const pkv_layer_t& L, int64_t tab, int j0, int nb) {
  uint32_t head = 0;
  int oldest = 0;
  for (int i = 0; i < nb; ++i) {
    const int j = j0 + i;
    const int64_t off = L.blk_off[tab + j];
    const uint32_t bytes = uint32_t((L.blk_len[tab + j] + 15) & ~15);
    const uint32_t size = bytes + 16;  // +16: slack for the decoders' word over-reads
    uint32_t pos = head % kRing;
    if (pos + size > kRing) {
      head += kRing - pos;
      pos = 0;
    }
    while (oldest < i && ((i - oldest) >= kTickets || head + size - R.abs[oldest % kTickets] > kRing)) {
      mbar_wait(&R.empty[oldest % kTickets], uint32_t((oldest / kTickets) & 1));
      ++oldest;
    }
    const int tk = i % kTickets;
    R.abs[tk] = head;
    R.start[tk] = pos;
    mbar_expect_tx(&R.full[tk], bytes);
    tma_load_1d(R.data + pos, L.arena + off, bytes, &R.full[tk]);
    head += size;
  }
}

// ======================================================================= V
// k-step ks of a block: k-slot 4t+e <-> (row-group t, token 8ks+e),
// 4t+16+e <-> (row-group t, token 8ks+4+e).  Lane (gi, tq) decodes whole packs
// of row-group tq and feeds tokens 0-7 to ks = 0 and 8-15 to ks = 1.
template <int NU>  // NU = unsigned digit tiles: 1 for G <= 4, 2 for G <= 8
__global__ void __launch_bounds__(kThreads) fused_v_i8_kernel(pkv_layer_t L, const float* __restrict__ w, int G,
                                                               int64_t wstride, float* __restrict__ part, int bpc,
                                                               int nsplit) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  uint8_t* rest = setup_ring(smem, R);
  uint32_t* desc_all = (uint32_t*)rest;                 // [kCW][512]
  float* vslow = (float*)(desc_all + kCW * 512);        // [kCW][8][kD] scalar-path partials
  float* sf = vslow + kCW * 8 * kD;                     // [8] fixed-point scale per head
  float* szs = sf + 8;                                  // [8] sum_t w*z per head
  float* red_w = szs + 8;                               // [kCW][8]
  float* red_s = red_w + kCW * 8;                       // [kCW]
  float* red_z = red_s + kCW;                           // [kCW][8]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int u = blockIdx.y, b = u / L.heads, h = u % L.heads, U = L.batch * L.heads;
  const int Hq = L.heads * G;
  const int nbk = L.nblk[b];
  const int j0 = blockIdx.x * bpc, j1 = min(nbk, j0 + bpc);
  const int nb = max(0, j1 - j0);
  const int64_t tab = (int64_t(1) * U + u) * L.max_blocks;
  const float* wu = w + (int64_t(b) * Hq + int64_t(h) * G) * wstride;
  for (int e = threadIdx.x; e < kCW * 8 * kD; e += blockDim.x) vslow[e] = 0.f;
  __syncthreads();

  if (warp == kCW) {
    if (lane == 0) produce(R, L, tab, j0, nb);
  }

  int accU[NU][8][4];
  int accS[8][4];
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      accS[mt][e] = 0;
#pragma unroll
      for (int nu = 0; nu < NU; ++nu) accU[nu][mt][e] = 0;
    }
  }

  if (warp < kCW) {
    // ---- pre-pass over the CTA's tokens (4 per step): max|w| per head, max scale, sum w*z
    const int tid = threadIdx.x;
    float wm[8], zs[8], smax = 0.f;
#pragma unroll
    for (int g = 0; g < 8; ++g) wm[g] = zs[g] = 0.f;
    for (int t4 = tid; t4 < nb * (kRows / 4); t4 += kCW * 32) {
      const int t = 4 * t4, j = j0 + t / kRows, r = t % kRows;
      const uint2* pp = (const uint2*)(L.arena + L.blk_off[tab + j] + kPar + 4 * r);
      const uint2 p01 = pp[0], p23 = pp[1];
      const float s4[4] = {h2f(p01.x & 0xffff), h2f(p01.y & 0xffff), h2f(p23.x & 0xffff), h2f(p23.y & 0xffff)};
      const float z4[4] = {h2f(p01.x >> 16), h2f(p01.y >> 16), h2f(p23.x >> 16), h2f(p23.y >> 16)};
      smax = fmaxf(smax, fmaxf(fmaxf(fabsf(s4[0]), fabsf(s4[1])), fmaxf(fabsf(s4[2]), fabsf(s4[3]))));
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        if (g < G) {
          const float4 wv = *(const float4*)(wu + int64_t(g) * wstride + int64_t(j) * kRows + r);
          wm[g] = fmaxf(wm[g], fmaxf(fmaxf(fabsf(wv.x), fabsf(wv.y)), fmaxf(fabsf(wv.z), fabsf(wv.w))));
          zs[g] = fmaf(wv.x, z4[0], fmaf(wv.y, z4[1], fmaf(wv.z, z4[2], fmaf(wv.w, z4[3], zs[g]))));
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      smax = fmaxf(smax, __shfl_xor_sync(PKV_FULL, smax, o));
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        wm[g] = fmaxf(wm[g], __shfl_xor_sync(PKV_FULL, wm[g], o));
        zs[g] += __shfl_xor_sync(PKV_FULL, zs[g], o);
      }
    }
    if (lane == 0) {
      red_s[warp] = smax;
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        red_w[warp * 8 + g] = wm[g];
        red_z[warp * 8 + g] = zs[g];
      }
    }
    consumer_sync();
    if (threadIdx.x < 8) {
      const int g = threadIdx.x;
      float m = 0.f, zz = 0.f, sm = 0.f;
      for (int wv = 0; wv < kCW; ++wv) {
        m = fmaxf(m, red_w[wv * 8 + g]);
        zz += red_z[wv * 8 + g];
        sm = fmaxf(sm, red_s[wv]);
      }
      const float v = m * sm;
      // |w * s * f| <= 2^22 so the 3-byte two's complement digits are exact
      float f = 1.f;
      if (v > 0.f) f = exp2f(fminf(fmaxf(floorf(log2f(4194304.f / v)), -120.f), 120.f));
      sf[g] = f;
      szs[g] = zz;
    }
    consumer_sync();

    // ---- main loop: this warp owns blocks warp, warp + kCW, ...
    uint32_t* desc = desc_all + warp * 512;
    float* vsl = vslow + warp * 8 * kD;
    const int gA = gi >> 1, gB = 4 + (gi >> 1);
    const float fA = sf[gA], fB = sf[gB];
    const uint32_t selU = uint32_t(gi & 1) | (uint32_t(4 + (gi & 1)) << 4);
    const uint32_t selS = 2u | (6u << 4);
    const bool odd = gi & 1;
    for (int i = warp; i < nb; i += kCW) {
      const int tk = i % kTickets;
      const int j = j0 + i;
      // weights of this lane's 16 tokens (row-group tq), issued before the wait
      float wa[16], wb[16];
      {
        const float* pa = wu + int64_t(gA) * wstride + int64_t(j) * kRows + 16 * tq;
        const float* pb = wu + int64_t(gB) * wstride + int64_t(j) * kRows + 16 * tq;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 va = make_float4(0.f, 0.f, 0.f, 0.f), vb = va;
          if (gA < G) va = *(const float4*)(pa + 4 * q);
          if (NU == 2 && gB < G) vb = *(const float4*)(pb + 4 * q);
          wa[4 * q] = va.x; wa[4 * q + 1] = va.y; wa[4 * q + 2] = va.z; wa[4 * q + 3] = va.w;
          wb[4 * q] = vb.x; wb[4 * q + 1] = vb.y; wb[4 * q + 2] = vb.z; wb[4 * q + 3] = vb.w;
        }
      }
      mbar_wait(&R.full[tk], uint32_t((i / kTickets) & 1));
      const uint8_t* blk = R.data + R.start[tk];
      const uint32_t* words = (const uint32_t*)blk;
      const bool fast = parse_block(blk, lane, desc);
      if (fast) {
        // B digits of x_t = rint(w_t * s_t * f) for the lane's 16 tokens
        uint32_t bu[NU][2][2], bs[2][2];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          uint32_t xa[8], xb[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int tok = 16 * tq + 8 * ks + 2 * q;
            const uint2 pr = *(const uint2*)(blk + kPar + 4 * tok);
            const float s0 = h2f(pr.x & 0xffff), s1 = h2f(pr.y & 0xffff);
            xa[2 * q] = uint32_t(__float2int_rn(wa[8 * ks + 2 * q] * fA * s0));
            xa[2 * q + 1] = uint32_t(__float2int_rn(wa[8 * ks + 2 * q + 1] * fA * s1));
            if (NU == 2) {
              xb[2 * q] = uint32_t(__float2int_rn(wb[8 * ks + 2 * q] * fB * s0));
              xb[2 * q + 1] = uint32_t(__float2int_rn(wb[8 * ks + 2 * q + 1] * fB * s1));
            }
          }
          bu[0][ks][0] = gather_byte(xa[0], xa[1], xa[2], xa[3], selU);
          bu[0][ks][1] = gather_byte(xa[4], xa[5], xa[6], xa[7], selU);
          if (NU == 2) {
            bu[NU - 1][ks][0] = gather_byte(xb[0], xb[1], xb[2], xb[3], selU);
            bu[NU - 1][ks][1] = gather_byte(xb[4], xb[5], xb[6], xb[7], selU);
            // S tile: column 2t -> head t (digit 2), 2t+1 -> head t+4
            bs[ks][0] = gather_byte(odd ? xb[0] : xa[0], odd ? xb[1] : xa[1], odd ? xb[2] : xa[2], odd ? xb[3] : xa[3], selS);
            bs[ks][1] = gather_byte(odd ? xb[4] : xa[4], odd ? xb[5] : xa[5], odd ? xb[6] : xa[6], odd ? xb[7] : xa[7], selS);
          } else {
            // S tile: column 2t -> head t (digit 2), 2t+1 -> zero
            bs[ks][0] = odd ? 0u : gather_byte(xa[0], xa[1], xa[2], xa[3], selS);
            bs[ks][1] = odd ? 0u : gather_byte(xa[4], xa[5], xa[6], xa[7], selS);
          }
        }
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int c = 16 * mt + gi;
          uint32_t P[4], Q[4];
          decode16(words, desc[tq * 128 + c], P);
          decode16(words, desc[tq * 128 + c + 8], Q);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t a[4] = {P[2 * ks], Q[2 * ks], P[2 * ks + 1], Q[2 * ks + 1]};
#pragma unroll
            for (int nu = 0; nu < NU; ++nu) imma_uu(accU[nu][mt], a, bu[nu][ks][0], bu[nu][ks][1]);
            imma_us(accS[mt], a, bs[ks][0], bs[ks][1]);
          }
        }
      } else {
        // scalar path: lane owns channels lane + 32q, all 64 tokens, all heads
        for (int r = 0; r < kRows; ++r) {
          const uint32_t pr = *(const uint32_t*)(blk + kPar + 4 * r);
          const float s = h2f(pr & 0xffff);
          float ws[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) ws[g] = g < G ? wu[int64_t(g) * wstride + int64_t(j) * kRows + r] * s : 0.f;
          const int rg = r >> 4, tt = r & 15;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = lane + 32 * q;
            const uint32_t d = desc[rg * 128 + c];
            const uint32_t wd = (d >> 18) & 15u;
            const float code = float(pack_min(blk, rg * 128 + c) + field_bytes(blk, (d & 0x3ffffu) + tt * wd, wd));
#pragma unroll
            for (int g = 0; g < 8; ++g) vsl[g * kD + c] = fmaf(ws[g], code, vsl[g * kD + c]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty[tk]);
    }
  }

  // ---- cross-warp reduction (fixed order), after every consumer finished
  __syncthreads();
  float* red = (float*)smem;  // [kCW][8][kD] (reuses the ring)
  if (warp < kCW) {
    const float* vsl = vslow + warp * 8 * kD;
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[(warp * 8 + g) * kD + lane + 32 * q] = vsl[g * kD + lane + 32 * q];
  }
  __syncthreads();
  if (warp < kCW) {
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int c = 16 * mt + gi + 8 * half;
        // tile U0: cols 2tq, 2tq+1 = head tq digits 0, 1; tile S col 2tq = head tq digit 2
        {
          const int g = tq;
          if (g < G) {
            const double v = double(accU[0][mt][2 * half]) + 256.0 * double(accU[0][mt][2 * half + 1]) +
                             65536.0 * double(accS[mt][2 * half]);
            red[(warp * 8 + g) * kD + c] += float(v / double(sf[g]));
          }
        }
        if (NU == 2) {
          const int g = tq + 4;
          if (g < G) {
            const double v = double(accU[NU - 1][mt][2 * half]) + 256.0 * double(accU[NU - 1][mt][2 * half + 1]) +
                             65536.0 * double(accS[mt][2 * half + 1]);
            red[(warp * 8 + g) * kD + c] += float(v / double(sf[g]));
          }
        }
      }
    }
  }
  __syncthreads();
  const int nr = (blockIdx.x == 0) ? L.nres[b] : 0;
  const uint16_t* vr = L.stage + (int64_t(1) * U + u) * L.buffer * kD;
  for (int e = threadIdx.x; e < G * (kD + 1); e += blockDim.x) {
    const int g = e / (kD + 1), c = e % (kD + 1);
    float s = 0.f;
    if (c < kD) {
#pragma unroll
      for (int wv = 0; wv < kCW; ++wv) s += red[(wv * 8 + g) * kD + c];
      const float* wr = wu + int64_t(g) * wstride + int64_t(nbk) * kRows;
      for (int t = 0; t < nr; ++t) s = fmaf(wr[t], __half2float(__ushort_as_half(vr[t * kD + c])), s);
    } else {
      s = szs[g];
    }
    part[((int64_t(u) * nsplit + blockIdx.x) * G + g) * (kD + 1) + c] = s;
  }
}

__global__ void fused_v_i8_finalize(const float* __restrict__ part, int U, int G, int nsplit, float* __restrict__ out) {
  const int64_t total = int64_t(U) * G * kD;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(e % kD);
    const int64_t ug = e / kD;
    const int gq = int(ug % G);
    const int64_t uu = ug / G;
    float s = 0.f, z = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float* pp = part + ((uu * nsplit + sp) * G + gq) * (kD + 1);
      s += pp[c];
      z += pp[kD];
    }
    out[e] = s + z;
  }
}

// ======================================================================= K
// Compute step m of a row-group covers K-layout positions 32m .. 32m+31:
// position 32m + 8s + n  <->  (column n of the 8-column tiles, channel select s).
// Lane (gi, tq) decodes the whole pack at position 32m + 8tq + gi.
// Transposition B1 k-slots: 4t+e <-> (select t, token e), 4t+16+e <-> (t, 4+e)
// within each 8-token half; A1 row r <-> (token r & 7, select sbase + (r >> 3)).
__device__ __forceinline__ uint32_t perm_byte(int row, int kappa, int sbase) {
  const int tqo = (kappa & 15) >> 2, e = kappa & 3, hi = kappa >> 4;
  return (tqo == sbase + (row >> 3)) && (4 * hi + e == (row & 7)) ? 1u : 0u;
}
// compute k2-slot -> physical K-layout position within the row-group
__device__ __forceinline__ int kslot_pos(int m, int slot) {
  const int hi = slot >> 4, tqo = (slot & 15) >> 2, e = slot & 3;
  const int n = 2 * tqo + (e & 1), s = 2 * hi + (e >> 1);
  return 32 * m + 8 * s + n;
}

template <int NU>
__global__ void __launch_bounds__(kThreads) fused_k_i8_kernel(pkv_layer_t L, const float* __restrict__ q, int G,
                                                               float* __restrict__ scores, int64_t sstride, int bpc) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  uint8_t* rest = setup_ring(smem, R);
  uint32_t* desc_all = (uint32_t*)rest;        // [kCW][512]
  float* sq = (float*)(desc_all + kCW * 512);  // [8][kD]
  float* sqsum = sq + 8 * kD;                  // [8]
  float* sfq = sqsum + 8;                      // [8]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int u = blockIdx.y, b = u / L.heads, h = u % L.heads, U = L.batch * L.heads;
  const int Hq = L.heads * G;
  const int nbk = L.nblk[b];
  const int j0 = blockIdx.x * bpc, j1 = min(nbk, j0 + bpc);
  const int nb = max(0, j1 - j0);
  const int64_t tab = (int64_t(0) * U + u) * L.max_blocks;
  float* srow = scores + (int64_t(b) * Hq + int64_t(h) * G) * sstride;
  const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * kD;
  for (int e = threadIdx.x; e < 8 * kD; e += blockDim.x) sq[e] = (e / kD) < G ? qu[e] : 0.f;
  __syncthreads();

  if (warp < kCW) {
    for (int g = warp; g < 8; g += kCW) {
      float s = 0.f, m = 0.f;
      for (int c = lane; c < kD; c += 32) {
        s += sq[g * kD + c];
        m = fmaxf(m, fabsf(sq[g * kD + c]));
      }
      s = warp_sum(s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(PKV_FULL, m, o));
      if (lane == 0) {
        sqsum[g] = s;
        sfq[g] = m > 0.f ? exp2f(fminf(fmaxf(floorf(log2f(4194304.f / m)), -120.f), 120.f)) : 1.f;
      }
    }
  }
  __syncthreads();
  if (warp == kCW) {  // producer; no CTA-wide barrier follows
    if (lane == 0) produce(R, L, tab, j0, nb);
    return;
  }

  // query digit fragments (B of the compute IMMA): col gi of tile U = (head gi/2, digit gi&1),
  // tile S col 2t = (head t, digit 2), col 2t+1 = (head t+4, digit 2) or zero
  uint32_t bqu[NU][4][2], bqs[4][2];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      uint32_t xu[NU][4], xs[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = kpos_to_col(kslot_pos(m, 4 * tq + 16 * r + e), kD);
#pragma unroll
        for (int nu = 0; nu < NU; ++nu) {
          const int g = 4 * nu + (gi >> 1);
          const int xi = __float2int_rn(sq[g * kD + c] * sfq[g]);
          xu[nu][e] = (uint32_t(xi) >> (8 * (gi & 1))) & 0xffu;
        }
        const int gs = (gi >> 1) + 4 * (gi & 1);
        const bool use = (gi & 1) == 0 || NU == 2;
        const int xi = __float2int_rn(sq[gs * kD + c] * sfq[gs]);
        xs[e] = use ? ((uint32_t(xi) >> 16) & 0xffu) : 0u;
      }
#pragma unroll
      for (int nu = 0; nu < NU; ++nu) bqu[nu][m][r] = xu[nu][0] | (xu[nu][1] << 8) | (xu[nu][2] << 16) | (xu[nu][3] << 24);
      bqs[m][r] = xs[0] | (xs[1] << 8) | (xs[2] << 16) | (xs[3] << 24);
    }
  }
  // transposition permutations: A1 for selects (0,1) and (2,3)
  uint32_t ap[2][4];
#pragma unroll
  for (int sb = 0; sb < 2; ++sb) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int row = gi + 8 * (r & 1);
      const int kb = 4 * tq + 16 * (r >> 1);
      ap[sb][r] = perm_byte(row, kb, 2 * sb) | (perm_byte(row, kb + 1, 2 * sb) << 8) |
                  (perm_byte(row, kb + 2, 2 * sb) << 16) | (perm_byte(row, kb + 3, 2 * sb) << 24);
    }
  }
  const float qs0 = sqsum[tq], fq0 = sfq[tq];
  const float qs1 = sqsum[(tq + 4) & 7], fq1 = sfq[(tq + 4) & 7];

  uint32_t* desc = desc_all + warp * 512;
  for (int i = warp; i < nb; i += kCW) {
    const int tk = i % kTickets;
    const int j = j0 + i;
    mbar_wait(&R.full[tk], uint32_t((i / kTickets) & 1));
    const uint8_t* blk = R.data + R.start[tk];
    const uint32_t* words = (const uint32_t*)blk;
    const bool fast = parse_block(blk, lane, desc);
    if (fast) {
#pragma unroll 1
      for (int rg = 0; rg < 4; ++rg) {
        int accU[NU][4], accS[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          accS[e] = 0;
#pragma unroll
          for (int nu = 0; nu < NU; ++nu) accU[nu][e] = 0;
        }
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          uint32_t P[4];
          decode16(words, desc[rg * 128 + 32 * m + 8 * tq + gi], P);
          int d[4][4];  // [token half a/b][select pair lo/hi]
          imma_uu0(d[0], ap[0], P[0], P[1]);  // tokens 0-7, selects 0/1
          imma_uu0(d[1], ap[1], P[0], P[1]);  // tokens 0-7, selects 2/3
          imma_uu0(d[2], ap[0], P[2], P[3]);  // tokens 8-15, selects 0/1
          imma_uu0(d[3], ap[1], P[2], P[3]);  // tokens 8-15, selects 2/3
          uint32_t a[4];
#pragma unroll
          for (int t = 0; t < 4; ++t)
            a[t] = uint32_t(d[(t & 1) * 2 + (t >> 1)][0]) | (uint32_t(d[(t & 1) * 2 + (t >> 1)][1]) << 8) |
                   (uint32_t(d[(t & 1) * 2 + (t >> 1)][2]) << 16) | (uint32_t(d[(t & 1) * 2 + (t >> 1)][3]) << 24);
#pragma unroll
          for (int nu = 0; nu < NU; ++nu) imma_uu(accU[nu], a, bqu[nu][m][0], bqu[nu][m][1]);
          imma_us(accS, a, bqs[m][0], bqs[m][1]);
        }
        const int tA = 16 * rg + gi, tB = tA + 8;
        const uint32_t pA = *(const uint32_t*)(blk + kPar + 4 * tA);
        const uint32_t pB = *(const uint32_t*)(blk + kPar + 4 * tB);
        const float sA = h2f(pA & 0xffff), zA = h2f(pA >> 16), sB = h2f(pB & 0xffff), zB = h2f(pB >> 16);
        if (tq < G) {
          const float vA = float(accU[0][0]) + 256.f * float(accU[0][1]) + 65536.f * float(accS[0]);
          const float vB = float(accU[0][2]) + 256.f * float(accU[0][3]) + 65536.f * float(accS[2]);
          srow[int64_t(tq) * sstride + int64_t(j) * kRows + tA] = fmaf(sA, vA / fq0, zA * qs0);
          srow[int64_t(tq) * sstride + int64_t(j) * kRows + tB] = fmaf(sB, vB / fq0, zB * qs0);
        }
        if (NU == 2 && tq + 4 < G) {
          const float vA = float(accU[NU - 1][0]) + 256.f * float(accU[NU - 1][1]) + 65536.f * float(accS[1]);
          const float vB = float(accU[NU - 1][2]) + 256.f * float(accU[NU - 1][3]) + 65536.f * float(accS[3]);
          srow[int64_t(tq + 4) * sstride + int64_t(j) * kRows + tA] = fmaf(sA, vA / fq1, zA * qs1);
          srow[int64_t(tq + 4) * sstride + int64_t(j) * kRows + tB] = fmaf(sB, vB / fq1, zB * qs1);
        }
      }
    } else {
      // scalar path: lane computes tokens lane and lane+32 for every head
      for (int half = 0; half < 2; ++half) {
        const int t = lane + 32 * half, rg = t >> 4, tt = t & 15;
        float acc[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) acc[g] = 0.f;
        for (int pos = 0; pos < 128; ++pos) {
          const uint32_t d = desc[rg * 128 + pos];
          const uint32_t wd = (d >> 18) & 15u;
          const float code = float(pack_min(blk, rg * 128 + pos) + field_bytes(blk, (d & 0x3ffffu) + tt * wd, wd));
          const int c = kpos_to_col(pos, kD);
#pragma unroll
          for (int g = 0; g < 8; ++g) acc[g] = fmaf(code, sq[g * kD + c], acc[g]);
        }
        const uint32_t pr = *(const uint32_t*)(blk + kPar + 4 * t);
        const float s = h2f(pr & 0xffff), z = h2f(pr >> 16);
        for (int g = 0; g < G; ++g) srow[int64_t(g) * sstride + int64_t(j) * kRows + t] = fmaf(s, acc[g], z * sqsum[g]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&R.empty[tk]);
  }

  if (blockIdx.x == 0) {  // uncompressed residue, same launch
    const int nr = L.nres[b];
    const uint16_t* kr = L.stage + (int64_t(0) * U + u) * L.buffer * kD;
    for (int t = warp; t < nr; t += kCW) {
      for (int g = 0; g < G; ++g) {
        float a = 0.f;
        for (int c = lane; c < kD; c += 32) a = fmaf(__half2float(__ushort_as_half(kr[t * kD + c])), sq[g * kD + c], a);
        a = warp_sum(a);
        if (lane == 0) srow[int64_t(g) * sstride + int64_t(nbk) * kRows + t] = a;
      }
    }
  }
}

constexpr size_t k_smem_bytes() { return kRingBytes + kCW * 512 * 4 + (8 * kD + 16) * 4; }
constexpr size_t v_smem_bytes() {
  const size_t a = kRingBytes + kCW * 512 * 4 + (kCW * 8 * kD + 8 + 8 + kCW * 8 + kCW + kCW * 8) * 4;
  const size_t r = size_t(kCW) * 8 * kD * 4;
  return a > r ? a : r;
}

}  // namespace

bool pkv_i8_supported(const pkv_layer_t* L, int G, int64_t stride) {
  return L->pack_size == kP && L->head_dim == kD && L->block == kRows && G >= 1 && G <= 8 && stride % 4 == 0;
}

int pkv_i8_fused_k(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
                   cudaStream_t s) {
  const size_t smem = k_smem_bytes();
  dim3 grid(max(1, (nblocks + kBpc - 1) / kBpc), L->batch * L->heads);
  if (G <= 4) {
    cudaFuncSetAttribute(fused_k_i8_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    fused_k_i8_kernel<1><<<grid, kThreads, smem, s>>>(*L, q, G, scores, sstride, kBpc);
  } else {
    cudaFuncSetAttribute(fused_k_i8_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    fused_k_i8_kernel<2><<<grid, kThreads, smem, s>>>(*L, q, G, scores, sstride, kBpc);
  }
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_k_scores(i8)");
}

int pkv_i8_fused_v(const pkv_layer_t* L, int nblocks, const float* w, int G, int64_t wstride, float* out,
                   float* part, cudaStream_t s) {
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  dim3 grid(nsplit, L->batch * L->heads);
  const size_t smem = v_smem_bytes();
  if (G <= 4) {
    cudaFuncSetAttribute(fused_v_i8_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    fused_v_i8_kernel<1><<<grid, kThreads, smem, s>>>(*L, w, G, wstride, part, kBpc, nsplit);
  } else {
    cudaFuncSetAttribute(fused_v_i8_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    fused_v_i8_kernel<2><<<grid, kThreads, smem, s>>>(*L, w, G, wstride, part, kBpc, nsplit);
  }
  const int64_t total = int64_t(L->batch) * L->heads * G * kD;
  const int fgrid = int((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  fused_v_i8_finalize<<<fgrid, 256, 0, s>>>(part, L->batch * L->heads, G, nsplit, out);
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_v_output(i8)");
}
