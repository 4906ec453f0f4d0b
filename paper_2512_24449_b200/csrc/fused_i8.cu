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

// D = A(u8) * B(s8), C = 0
__device__ __forceinline__ void imma_us0(int (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};\n"
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

// a*b + c forced onto the FMA pipe (IMAD), keeping the ALU pipe for byte work
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Four fields at stride w (w <= 4) in the low bits of x -> one byte each,
// plus the pack minimum: exact uint8 codes (byte e = field e).  Left shifts
// are multiplies by M1 = 2^(16-2w) / M2 = 2^(8-w) (FMA pipe); the byte
// permutes and the mask stay on the ALU pipe.
__device__ __forceinline__ uint32_t spread4(uint32_t x, uint32_t M1, uint32_t M2, uint32_t m4, uint32_t mr) {
  const uint32_t y = __byte_perm(x, x * M1, 0x7610);  // fields 0,1 low half; 2,3 high half
  const uint32_t z = __byte_perm(y, y * M2, 0x7250);  // one field per byte
  return imad(z & m4, 1u, mr);
}

// All 16 fields of the pack described by `d` (w <= 4) as uint8 codes:
// r[q] holds tokens 4q..4q+3 (byte e = token 4q+e).
__device__ __forceinline__ void decode16(const uint32_t* __restrict__ words, uint32_t d, uint32_t (&r)[4]) {
  const uint32_t bo = d & 0x3ffffu;
  const uint32_t w = (d >> 18) & 15u;
  const uint32_t* p = words + (bo >> 5);
  const uint32_t w0 = p[0], w1 = p[1], w2 = p[2];
  const uint32_t xlo = __funnelshift_r(w0, w1, bo);   // payload bits 0..31
  const uint32_t xmid = __funnelshift_r(w1, w2, bo);  // payload bits 32..63
  const uint32_t M2 = 256u >> w, M1 = M2 * M2, M3 = M1 * M1;  // 2^(8-w), 2^(16-2w), 2^(32-4w)
  const uint32_t xhi = __funnelshift_rc(xlo, xmid, w * 8u);    // fields 8..15
  const uint32_t m4 = imad(0x01010101u, 1u << w, 0u - 0x01010101u);
  const uint32_t mr = (d >> 22) * 0x01010101u;
  r[0] = spread4(xlo, M1, M2, m4, mr);
  r[1] = spread4(__umulhi(xlo, M3), M1, M2, m4, mr);  // x >> 4w on the FMA pipe
  r[2] = spread4(xhi, M1, M2, m4, mr);
  r[3] = spread4(__umulhi(xhi, M3), M1, M2, m4, mr);
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
// Persistent CTAs: work item = (unit, split of <= kBpc blocks); CTA c owns items
// c, c + gridDim.x, ...  The producer warp streams the blocks of all its items
// back to back through the byte ring (tickets are global across items), so the
// ring never drains at item boundaries.
struct Ring {
  uint8_t* data;
  uint64_t* full;
  uint64_t* empty;
  uint32_t* start;  // [kTickets] ring offset of each ticket's block
  uint32_t* abs;    // [kTickets] producer-private absolute start
  int64_t* soff;    // [kBpc] producer-private block offsets of the current item
  int* slen;        // [kBpc]
};
constexpr size_t kRingBytes = kRing + kTickets * 16 + kTickets * 8 + kBpc * 12;

__device__ __forceinline__ uint8_t* setup_ring(uint8_t* smem, Ring& R) {
  R.data = smem;
  R.full = (uint64_t*)(smem + kRing);
  R.empty = R.full + kTickets;
  R.start = (uint32_t*)(R.empty + kTickets);
  R.abs = R.start + kTickets;
  R.soff = (int64_t*)(R.abs + kTickets);
  R.slen = (int*)(R.soff + kBpc);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTickets; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], 1);
    }
    fence_barrier_init();
  }
  return smem + kRingBytes;
}

struct Item {
  int u, s, b, h, j0, nb, nbk;
};
__device__ __forceinline__ Item item_of(const pkv_layer_t& L, int item, int nsplit) {
  Item it;
  it.u = item / nsplit;
  it.s = item - it.u * nsplit;
  it.b = it.u / L.heads;
  it.h = it.u - it.b * L.heads;
  it.nbk = L.nblk[it.b];
  it.j0 = it.s * kBpc;
  it.nb = max(0, min(kBpc, it.nbk - it.j0));
  return it;
}

// Producer warp: for every item of this CTA, stage its block table in smem
// (warp-parallel), then one lane issues the TMA copies.
__device__ void produce(const Ring& R, const pkv_layer_t& L, int kind, int nsplit, int nitems, int lane) {
  const int U = L.batch * L.heads;
  uint32_t head = 0;
  int oldest = 0, ticket = 0;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const Item it = item_of(L, item, nsplit);
    const int64_t tab = (int64_t(kind) * U + it.u) * L.max_blocks + it.j0;
    if (lane < it.nb) {
      R.soff[lane] = L.blk_off[tab + lane];
      R.slen[lane] = L.blk_len[tab + lane];
    }
    __syncwarp();
    if (lane == 0) {
      for (int i = 0; i < it.nb; ++i, ++ticket) {
        const uint32_t bytes = uint32_t((R.slen[i] + 15) & ~15);
        const uint32_t size = bytes + 16;  // +16: slack for the decoders' word over-reads
        uint32_t pos = head % kRing;
        if (pos + size > kRing) {
          head += kRing - pos;
          pos = 0;
        }
        while (oldest < ticket &&
               ((ticket - oldest) >= kTickets || head + size - R.abs[oldest % kTickets] > kRing)) {
          mbar_wait(&R.empty[oldest % kTickets], uint32_t((oldest / kTickets) & 1));
          ++oldest;
        }
        const int tk = ticket % kTickets;
        R.abs[tk] = head;
        R.start[tk] = pos;
        mbar_expect_tx(&R.full[tk], bytes);
        tma_load_1d(R.data + pos, L.arena + R.soff[i], bytes, &R.full[tk]);
        head += size;
      }
    }
    __syncwarp();
  }
}

// ======================================================================= V
// k-step ks of a block: k-slot 4t+e <-> (row-group t, token 8ks+e),
// 4t+16+e <-> (row-group t, token 8ks+4+e).  Lane (gi, tq) decodes whole packs
// of row-group tq and feeds tokens 0-7 to ks = 0 and 8-15 to ks = 1.
// B = digits of x_t = rint(w_t * s_t * f), f a power of two chosen per block
// and head so |x| <= 2^22; the int32 tile sums of each block are converted to
// f32 (divided by f) into per-lane float accumulators.
template <int NU>  // NU = unsigned digit tiles: 1 for G <= 4, 2 for G <= 8
__global__ void __launch_bounds__(kThreads) fused_v_i8_kernel(pkv_layer_t L, const float* __restrict__ w, int G,
                                                               int64_t wstride, float* __restrict__ part, int nsplit,
                                                               int nitems, float* __restrict__ vscr) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  uint8_t* rest = setup_ring(smem, R);
  uint32_t* desc_all = (uint32_t*)rest;                 // [kCW][512]
  float* red = (float*)(desc_all + kCW * 512);          // [kCW][8][kD]
  float* zred = red + kCW * 8 * kD;                     // [kCW][8]
  int* touched = (int*)(zred + kCW * 8);                // [kCW]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int U = L.batch * L.heads;
  if (threadIdx.x < kCW) touched[threadIdx.x] = 0;
  __syncthreads();
  if (warp == kCW) {  // producer; no CTA-wide barrier follows
    produce(R, L, 1, nsplit, nitems, lane);
    return;
  }

  uint32_t* desc = desc_all + warp * 512;
  float* vsl = vscr + (int64_t(blockIdx.x) * kCW + warp) * (8 * kD);  // scalar-path partials
  const int gA = gi >> 1, gB = 4 + (gi >> 1);
  const uint32_t selU = uint32_t(gi & 1) | (uint32_t(4 + (gi & 1)) << 4);
  const uint32_t selS = 2u | (6u << 4);
  const bool odd = gi & 1;
  int ticket_base = 0;

#pragma unroll 1
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const Item it = item_of(L, item, nsplit);
    const int Hq = L.heads * G;
    const float* wu = w + (int64_t(it.b) * Hq + int64_t(it.h) * G) * wstride;
    float accF[NU][8][2];
#pragma unroll
    for (int nu = 0; nu < NU; ++nu)
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) accF[nu][mt][0] = accF[nu][mt][1] = 0.f;
    float zacc[NU] = {};
    bool slow_used = false;

#pragma unroll 1
    for (int i = warp; i < it.nb; i += kCW) {
      const int t = ticket_base + i;
      const int tk = t % kTickets;
      const int j = it.j0 + i;
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
      mbar_wait(&R.full[tk], uint32_t((t / kTickets) & 1));
      const uint8_t* blk = R.data + R.start[tk];
      const uint32_t* words = (const uint32_t*)blk;
      // w*s and w*z for the lane's tokens
      float mA = 0.f, mB = 0.f;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint2 pr = *(const uint2*)(blk + kPar + 4 * (16 * tq + 2 * q));
        const float s0 = h2f(pr.x & 0xffff), s1 = h2f(pr.y & 0xffff);
        const float z0 = h2f(pr.x >> 16), z1 = h2f(pr.y >> 16);
        if (!odd) {  // one lane per (head, row-group) adds the z term
          zacc[0] = fmaf(wa[2 * q], z0, fmaf(wa[2 * q + 1], z1, zacc[0]));
          if (NU == 2) zacc[NU - 1] = fmaf(wb[2 * q], z0, fmaf(wb[2 * q + 1], z1, zacc[NU - 1]));
        }
        wa[2 * q] *= s0;
        wa[2 * q + 1] *= s1;
        mA = fmaxf(mA, fmaxf(fabsf(wa[2 * q]), fabsf(wa[2 * q + 1])));
        if (NU == 2) {
          wb[2 * q] *= s0;
          wb[2 * q + 1] *= s1;
          mB = fmaxf(mB, fmaxf(fabsf(wb[2 * q]), fabsf(wb[2 * q + 1])));
        }
      }
      // block max per head: lanes (gi, tq) with the same gi >> 1
#pragma unroll
      for (int o = 1; o <= 4; o <<= 1) {
        mA = fmaxf(mA, __shfl_xor_sync(PKV_FULL, mA, o));
        if (NU == 2) mB = fmaxf(mB, __shfl_xor_sync(PKV_FULL, mB, o));
      }
      const float fA = mA > 0.f ? exp2f(fminf(floorf(log2f(4194304.f / mA)), 120.f)) : 1.f;
      const float fB = mB > 0.f ? exp2f(fminf(floorf(log2f(4194304.f / mB)), 120.f)) : 1.f;
      const bool fast = parse_block(blk, lane, desc);
      if (fast) {
        uint32_t bu[NU][2][2], bs[2][2];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          uint32_t xa[8], xb[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            xa[e] = uint32_t(__float2int_rn(wa[8 * ks + e] * fA));
            if (NU == 2) xb[e] = uint32_t(__float2int_rn(wb[8 * ks + e] * fB));
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
            bs[ks][0] = odd ? 0u : gather_byte(xa[0], xa[1], xa[2], xa[3], selS);
            bs[ks][1] = odd ? 0u : gather_byte(xa[4], xa[5], xa[6], xa[7], selS);
          }
        }
        // inverse scales of the heads this lane's D columns belong to (head tq, tq + 4)
        const float inv0 = 1.f / __shfl_sync(PKV_FULL, fA, (2 * tq) << 2);
        const float inv1 = NU == 2 ? 1.f / __shfl_sync(PKV_FULL, fB, (2 * tq) << 2) : 0.f;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int c = 16 * mt + gi;
          uint32_t P[4], Q[4];
          decode16(words, desc[tq * 128 + c], P);
          decode16(words, desc[tq * 128 + c + 8], Q);
          int dU[NU][4], dS[4];
          {
            const uint32_t a[4] = {P[0], Q[0], P[1], Q[1]};
#pragma unroll
            for (int nu = 0; nu < NU; ++nu) imma_uu0(dU[nu], a, bu[nu][0][0], bu[nu][0][1]);
            imma_us0(dS, a, bs[0][0], bs[0][1]);
          }
          {
            const uint32_t a[4] = {P[2], Q[2], P[3], Q[3]};
#pragma unroll
            for (int nu = 0; nu < NU; ++nu) imma_uu(dU[nu], a, bu[nu][1][0], bu[nu][1][1]);
            imma_us(dS, a, bs[1][0], bs[1][1]);
          }
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            accF[0][mt][half] = fmaf(float(dU[0][2 * half]) + 256.f * float(dU[0][2 * half + 1]) +
                                         65536.f * float(dS[2 * half]), inv0, accF[0][mt][half]);
            if (NU == 2)
              accF[NU - 1][mt][half] = fmaf(float(dU[NU - 1][2 * half]) + 256.f * float(dU[NU - 1][2 * half + 1]) +
                                                65536.f * float(dS[2 * half + 1]), inv1, accF[NU - 1][mt][half]);
          }
        }
      } else {
        // scalar path (rare): lane owns channels lane + 32q, all 64 tokens, all heads;
        // partials accumulate in this warp's global scratch (fixed order, deterministic)
        if (!slow_used) {
          for (int e = lane; e < 8 * kD; e += 32) vsl[e] = 0.f;
          __syncwarp();
          slow_used = true;
        }
        float acc[8][4];
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[g][q] = vsl[g * kD + lane + 32 * q];
#pragma unroll 1
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
            for (int g = 0; g < 8; ++g) acc[g][q] = fmaf(ws[g], code, acc[g][q]);
          }
        }
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
          for (int q = 0; q < 4; ++q) vsl[g * kD + lane + 32 * q] = acc[g][q];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty[tk]);
    }
    ticket_base += it.nb;

    // ---- item epilogue: fixed-order cross-warp reduction
#pragma unroll
    for (int nu = 0; nu < NU; ++nu) {
      zacc[nu] += __shfl_xor_sync(PKV_FULL, zacc[nu], 1);
      zacc[nu] += __shfl_xor_sync(PKV_FULL, zacc[nu], 2);
    }
    consumer_sync();  // previous item's readers of red are done
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[(warp * 8 + g) * kD + lane + 32 * q] = slow_used ? vsl[g * kD + lane + 32 * q] : 0.f;
    if (tq == 0 && !odd) {
      zred[warp * 8 + gA] = zacc[0];
      if (NU == 2) zred[warp * 8 + gB] = zacc[NU - 1];
    }
    if (tq == 0 && odd && NU == 1) zred[warp * 8 + 4 + gA] = 0.f;
    if (NU == 1 && lane < 4) zred[warp * 8 + 4 + lane] = 0.f;
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int c = 16 * mt + gi + 8 * half;
        red[(warp * 8 + tq) * kD + c] += accF[0][mt][half];
        if (NU == 2) red[(warp * 8 + tq + 4) * kD + c] += accF[NU - 1][mt][half];
      }
    }
    consumer_sync();
    const int nr = (it.s == 0) ? L.nres[it.b] : 0;
    const uint16_t* vr = L.stage + (int64_t(1) * U + it.u) * L.buffer * kD;
    for (int e = threadIdx.x; e < G * (kD + 1); e += kCW * 32) {
      const int g = e / (kD + 1), c = e % (kD + 1);
      float sum = 0.f;
      if (c < kD) {
#pragma unroll
        for (int wv = 0; wv < kCW; ++wv) sum += red[(wv * 8 + g) * kD + c];
        const float* wr = wu + int64_t(g) * wstride + int64_t(it.nbk) * kRows;
        for (int t = 0; t < nr; ++t) sum = fmaf(wr[t], __half2float(__ushort_as_half(vr[t * kD + c])), sum);
      } else {
#pragma unroll
        for (int wv = 0; wv < kCW; ++wv) sum += zred[wv * 8 + g];
      }
      part[((int64_t(it.u) * nsplit + it.s) * G + g) * (kD + 1) + c] = sum;
    }
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
                                                               float* __restrict__ scores, int64_t sstride,
                                                               int nsplit, int nitems) {
  extern __shared__ __align__(128) uint8_t smem[];
  Ring R;
  uint8_t* rest = setup_ring(smem, R);
  uint32_t* desc_all = (uint32_t*)rest;        // [kCW][512]
  float* sq = (float*)(desc_all + kCW * 512);  // [8][kD]
  float* sqsum = sq + 8 * kD;                  // [8]
  float* sfq = sqsum + 8;                      // [8]
  uint32_t* sbq = (uint32_t*)(sfq + 8);        // [8][NU+1][32] query digit fragments
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int U = L.batch * L.heads;
  __syncthreads();
  if (warp == kCW) {  // producer; no CTA-wide barrier follows
    produce(R, L, 0, nsplit, nitems, lane);
    return;
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
  uint32_t* desc = desc_all + warp * 512;
  const int tid = threadIdx.x;
  // query of the first item (next items are prefetched into registers)
  float qn[8];
  auto load_q = [&](int item) {
    const Item it = item_of(L, item, nsplit);
    const float* qu = q + (int64_t(it.b) * L.heads * G + int64_t(it.h) * G) * kD;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int e = tid + k * kCW * 32;
      qn[k] = (e / kD) < G ? qu[e] : 0.f;
    }
  };
  if (blockIdx.x < nitems) load_q(blockIdx.x);
  int ticket_base = 0;

#pragma unroll 1
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    const Item it = item_of(L, item, nsplit);
    const int Hq = L.heads * G;
    float* srow = scores + (int64_t(it.b) * Hq + int64_t(it.h) * G) * sstride;
    consumer_sync();  // every consumer is done with the previous item's query
#pragma unroll
    for (int k = 0; k < 8; ++k) sq[tid + k * kCW * 32] = qn[k];
    consumer_sync();
    if (item + int(gridDim.x) < nitems) load_q(item + gridDim.x);  // prefetch the next item's query
    for (int g = warp; g < 8; g += kCW) {
      float sm = 0.f, m = 0.f;
      for (int c = lane; c < kD; c += 32) {
        sm += sq[g * kD + c];
        m = fmaxf(m, fabsf(sq[g * kD + c]));
      }
      sm = warp_sum(sm);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(PKV_FULL, m, o));
      if (lane == 0) {
        sqsum[g] = sm;
        sfq[g] = m > 0.f ? exp2f(fminf(fmaxf(floorf(log2f(4194304.f / m)), -120.f), 120.f)) : 1.f;
      }
    }
    consumer_sync();
    // query digit fragments (B of the compute IMMA), built once per item in shared
    // memory by all consumer threads: col gi of tile U = (head gi/2, digit gi&1),
    // tile S col 2t = (head t, digit 2), col 2t+1 = (head t+4, digit 2) or zero
#pragma unroll 1
    for (int e = tid; e < 8 * (NU + 1) * 32; e += kCW * 32) {
      const int ln = e & 31, idx = e >> 5, tt = idx % (NU + 1), mr = idx / (NU + 1);
      const int m = mr >> 1, r = mr & 1, lgi = ln >> 2, ltq = ln & 3;
      uint32_t v = 0;
#pragma unroll 1
      for (int ee = 0; ee < 4; ++ee) {
        const int c = kpos_to_col(kslot_pos(m, 4 * ltq + 16 * r + ee), kD);
        uint32_t byte;
        if (tt < NU) {
          const int g = 4 * tt + (lgi >> 1);
          byte = (uint32_t(__float2int_rn(sq[g * kD + c] * sfq[g])) >> (8 * (lgi & 1))) & 0xffu;
        } else {
          const int gs = (lgi >> 1) + 4 * (lgi & 1);
          const bool use = (lgi & 1) == 0 || NU == 2;
          byte = use ? (uint32_t(__float2int_rn(sq[gs * kD + c] * sfq[gs])) >> 16) & 0xffu : 0u;
        }
        v |= byte << (8 * ee);
      }
      sbq[e] = v;
    }
    consumer_sync();
    uint32_t bqu[NU][4][2], bqs[4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
#pragma unroll
        for (int nu = 0; nu < NU; ++nu) bqu[nu][m][r] = sbq[((m * 2 + r) * (NU + 1) + nu) * 32 + lane];
        bqs[m][r] = sbq[((m * 2 + r) * (NU + 1) + NU) * 32 + lane];
      }
    const float qs0 = sqsum[tq], fq0 = 1.f / sfq[tq];
    const float qs1 = sqsum[(tq + 4) & 7], fq1 = 1.f / sfq[(tq + 4) & 7];

#pragma unroll 1
    for (int i = warp; i < it.nb; i += kCW) {
      const int t = ticket_base + i;
      const int tk = t % kTickets;
      const int j = it.j0 + i;
      mbar_wait(&R.full[tk], uint32_t((t / kTickets) & 1));
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
            for (int x4 = 0; x4 < 4; ++x4) {
              const int x = (x4 & 1) * 2 + (x4 >> 1);
              a[x4] = uint32_t(d[x][0]) | (uint32_t(d[x][1]) << 8) | (uint32_t(d[x][2]) << 16) | (uint32_t(d[x][3]) << 24);
            }
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
            srow[int64_t(tq) * sstride + int64_t(j) * kRows + tA] = fmaf(sA, vA * fq0, zA * qs0);
            srow[int64_t(tq) * sstride + int64_t(j) * kRows + tB] = fmaf(sB, vB * fq0, zB * qs0);
          }
          if (NU == 2 && tq + 4 < G) {
            const float vA = float(accU[NU - 1][0]) + 256.f * float(accU[NU - 1][1]) + 65536.f * float(accS[1]);
            const float vB = float(accU[NU - 1][2]) + 256.f * float(accU[NU - 1][3]) + 65536.f * float(accS[3]);
            srow[int64_t(tq + 4) * sstride + int64_t(j) * kRows + tA] = fmaf(sA, vA * fq1, zA * qs1);
            srow[int64_t(tq + 4) * sstride + int64_t(j) * kRows + tB] = fmaf(sB, vB * fq1, zB * qs1);
          }
        }
      } else {
        // scalar path (rare): lane computes tokens lane and lane+32 for every head
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          const int tt = lane + 32 * half, rg = tt >> 4, t16 = tt & 15;
          float acc[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) acc[g] = 0.f;
#pragma unroll 1
          for (int pos = 0; pos < 128; ++pos) {
            const uint32_t d = desc[rg * 128 + pos];
            const uint32_t wd = (d >> 18) & 15u;
            const float code = float(pack_min(blk, rg * 128 + pos) + field_bytes(blk, (d & 0x3ffffu) + t16 * wd, wd));
            const int c = kpos_to_col(pos, kD);
#pragma unroll
            for (int g = 0; g < 8; ++g) acc[g] = fmaf(code, sq[g * kD + c], acc[g]);
          }
          const uint32_t pr = *(const uint32_t*)(blk + kPar + 4 * tt);
          const float s = h2f(pr & 0xffff), z = h2f(pr >> 16);
          for (int g = 0; g < G; ++g) srow[int64_t(g) * sstride + int64_t(j) * kRows + tt] = fmaf(s, acc[g], z * sqsum[g]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&R.empty[tk]);
    }
    ticket_base += it.nb;
    if (it.s == 0) {  // uncompressed residue of this unit
      const int nr = L.nres[it.b];
      const uint16_t* kr = L.stage + (int64_t(0) * U + it.u) * L.buffer * kD;
      for (int t = warp; t < nr; t += kCW) {
        for (int g = 0; g < G; ++g) {
          float a = 0.f;
          for (int c = lane; c < kD; c += 32) a = fmaf(__half2float(__ushort_as_half(kr[t * kD + c])), sq[g * kD + c], a);
          a = warp_sum(a);
          if (lane == 0) srow[int64_t(g) * sstride + int64_t(it.nbk) * kRows + t] = a;
        }
      }
    }
  }
}

constexpr size_t k_smem_bytes() { return kRingBytes + kCW * 512 * 4 + (8 * kD + 16) * 4 + 8 * 3 * 32 * 4; }
constexpr size_t v_smem_bytes() { return kRingBytes + kCW * 512 * 4 + (kCW * 8 * kD + kCW * 8 + kCW) * 4; }

template <class K>
int persistent_grid(K kernel, size_t smem, int nitems) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kThreads, smem);
  return max(1, min(nitems, max(1, per) * nsm));
}

}  // namespace

bool pkv_i8_supported(const pkv_layer_t* L, int G, int64_t stride) {
  return L->pack_size == kP && L->head_dim == kD && L->block == kRows && G >= 1 && G <= 8 && stride % 4 == 0;
}

int pkv_i8_fused_k(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
                   cudaStream_t s) {
  const size_t smem = k_smem_bytes();
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  const int nitems = nsplit * L->batch * L->heads;
  if (G <= 4) {
    cudaFuncSetAttribute(fused_k_i8_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int grid = persistent_grid(fused_k_i8_kernel<1>, smem, nitems);
    fused_k_i8_kernel<1><<<grid, kThreads, smem, s>>>(*L, q, G, scores, sstride, nsplit, nitems);
  } else {
    cudaFuncSetAttribute(fused_k_i8_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int grid = persistent_grid(fused_k_i8_kernel<2>, smem, nitems);
    fused_k_i8_kernel<2><<<grid, kThreads, smem, s>>>(*L, q, G, scores, sstride, nsplit, nitems);
  }
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_k_scores(i8)");
}

int64_t pkv_i8_v_scratch(const pkv_layer_t* L, int nblocks, int G) {
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  const int64_t items = int64_t(nsplit) * L->batch * L->heads;
  return items * G * (kD + 1) * 4 + int64_t(148 * 8) * kCW * 8 * kD * 4;
}

int pkv_i8_fused_v(const pkv_layer_t* L, int nblocks, const float* w, int G, int64_t wstride, float* out,
                   float* part, cudaStream_t s) {
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  const int nitems = nsplit * L->batch * L->heads;
  const size_t smem = v_smem_bytes();
  float* vscr = part + int64_t(nitems) * G * (kD + 1);
  if (G <= 4) {
    cudaFuncSetAttribute(fused_v_i8_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int grid = min(persistent_grid(fused_v_i8_kernel<1>, smem, nitems), 148 * 8);
    fused_v_i8_kernel<1><<<grid, kThreads, smem, s>>>(*L, w, G, wstride, part, nsplit, nitems, vscr);
  } else {
    cudaFuncSetAttribute(fused_v_i8_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int grid = min(persistent_grid(fused_v_i8_kernel<2>, smem, nitems), 148 * 8);
    fused_v_i8_kernel<2><<<grid, kThreads, smem, s>>>(*L, w, G, wstride, part, nsplit, nitems, vscr);
  }
  const int64_t total = int64_t(L->batch) * L->heads * G * kD;
  const int fgrid = int((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  fused_v_i8_finalize<<<fgrid, 256, 0, s>>>(part, L->batch * L->heads, G, nsplit, out);
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_v_output(i8)");
}
