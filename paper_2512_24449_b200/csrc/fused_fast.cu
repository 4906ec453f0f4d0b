// fused_fast.cu — fused decompress + GEMV for the default format (pack size 16,
// head_dim 128, 64-token blocks), sm_100a.
//
// Warp-level persistent work split: warp W of the grid owns a contiguous,
// equal-sized range of the layer's (unit, block) sequence, unit = (sequence,
// kv-head).  Every warp is its own producer:
//  * it streams its blocks with 1-D TMA bulk copies (cp.async.bulk + mbarrier
//    complete_tx) into a private shared-memory byte ring (V: 11 KB, up to two
//    blocks ahead; K: 5.9 KB so 4 CTAs fit per SM, plus an L2 bulk prefetch
//    two blocks ahead).  Bulk copies issued by one warp are serviced one after
//    another, so a single producer warp per CTA cannot feed HBM-rate decoding.
//  * Lane l walks a run of physically consecutive packs (SPEC.md:330 payloads
//    are contiguous in physical pack order), so one warp prefix scan of the
//    width nibbles gives each lane its starting bit and the lane
//    then advances by 16*w bits per pack — no per-pack descriptor table.
//  * Unpack (pack size 16, width w <= 4): two funnel shifts extract the pack's
//    64-bit payload, the width's shift multipliers and byte mask come from a
//    16-entry shared-memory table (V) or registers (K), and a three-level
//    select tree places the 16
//    fields into 4 registers of 4 bytes with the pack minimum added, i.e. the
//    exact uint8 codes (SPEC.md:120 q values).  Byte order within a pack:
//    position m holds row tok(m) = m with bits 1 and 2 swapped.
//  * Products on the int8 tensor cores (mma.sync m16n8k32, IMMA).  The other
//    operand is exact fixed point: the query (K) in 3 byte digits (~23 bits),
//    w_t*scale_t (V, non-negative) in 2 unsigned byte digits scaled per block
//    and head, so every tile sum is exact in int32.
//  * K: the reduction runs over channels but packs run along
//    rows, so every lane stores its decoded packs (16 rows of one channel =
//    16 bytes) into a per-warp [row-group][channel][16] tile and
//    ldmatrix.m16n16.trans.b8 reads them back transposed as the A fragment.
//    score = s_t * (acc / 2^S) + z_t * sum(q)  (dequantisation factored).
//  * V: rows are the MMA k dimension, the pack direction, so
//    the decoded registers are the A fragment directly (no transpose).
//    out = sum_t (w_t s_t) code + sum_t w_t z_t.
// Blocks with packs of width 5..7 run a second, block-uniform unpack (four
// 4-field spreads per pack); blocks with a width >= 8 or a large minimum take a
// scalar path inside the same launch (never at the default rel 0.1 / 0.2).
#include "pkv_common.cuh"

#include <mutex>
#include <type_traits>
#include <vector>

using namespace pkv;

#include "fast_common.cuh"

namespace {

// ======================================================================= K
// Per-warp tile: [row-group g][channel c][16 bytes], row R = 128g + c at byte
// 16 * (R ^ (((R >> 6) & 1) << 2)) (XOR swizzle of the 16-byte chunk within a
// 128-byte line: each quarter-warp of a decode step's STS.128 and each 8-row
// phase of the ldmatrix hit 8 distinct chunks, i.e. no bank conflicts).
constexpr int kTile = 4 * 128 * 16;  // 8 KB
constexpr int kWK = 4;               // warps per CTA
// Diagnostic builds (tools/exp/build_variant.sh -D...; results are wrong, timing
// only): skip the unpack arithmetic, skip the MMA + epilogue, keep
// only the feed, or record per-warp feed-wait cycles into the scores buffer.
#ifndef PKV_DIAG_NODECODE
#define PKV_DIAG_NODECODE 0
#endif
#ifndef PKV_DIAG_NOMMA
#define PKV_DIAG_NOMMA 0
#endif
#ifndef PKV_DIAG_FEEDONLY
#define PKV_DIAG_FEEDONLY 0
#endif
#ifndef PKV_DIAG_WAITCLK
#define PKV_DIAG_WAITCLK 0
#endif
#ifndef PKV_DIAG_FEEDPARSE
#define PKV_DIAG_FEEDPARSE 0
#endif
#ifndef PKV_DIAG_NOSTS
#define PKV_DIAG_NOSTS 0
#endif
#ifndef PKV_RBK  // ring bytes / slots per K warp (-D overrides for tools/exp variants)
// 5.9 KB: 8 KB tile + ring fit 4 CTAs of 4 warps per SM (16 warps) and still
// hold the largest narrow-width block (w <= 4: 1544 + 512 * 8 B); a block with
// wider packs (w 5..7, up to ~8.7 KB) that does not fit is decoded in place
// from global memory (same fast path, global loads); measured 67.3 us vs
// 69.8 us for a 10 KB ring at 3 CTAs per SM (config B)
#define PKV_RBK 5888
#endif
#ifndef PKV_KRR
#define PKV_KRR 0
#endif
#ifndef PKV_KMINB  // K: CTAs per SM the register allocation must allow (1: no bound)
// 4: <= 128 registers, so the score-statistics (ST, attention) and G <= 8 instantiations
// (132 / 141-147 registers unbounded, 3 CTAs per SM) also run 4 CTAs = 16 warps per SM, as
// the shared memory allows: config B three-launch attention 132.0 -> 128.4 us, config E
// fused K 486 -> 466 us, attention 1026 -> 1009 us (same box, kbench)
#define PKV_KMINB 4
#endif
#ifndef PKV_NSK
#define PKV_NSK 3
#endif
constexpr int kRBK = PKV_RBK, kNSK = PKV_NSK;
using FeedK = Feed<kRBK, kNSK>;
constexpr size_t kWarpSmemK = (kTile + FeedK::bytes() + 127) / 128 * 128;



// ST: also record softmax statistics for attention_decode: the maximum score of
// every (unit, warp slot, head) in kmax[u][slot][g] and of the residue rows in
// kres[u][g] (-inf when there are none).
template <int NU, bool ST>  // NU: unsigned query digit tiles, 1 for G <= 4, 2 for G <= 8
__global__ void __launch_bounds__(kWK * 32, PKV_KMINB) fused_k_fast_kernel(pkv_layer_t L, const float* __restrict__ q, int G,
                                                                 float* __restrict__ scores, int64_t sstride, int NB,
                                                                 int64_t total, float* __restrict__ kmax,
                                                                 float* __restrict__ kres, int kslots) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int U = L.batch * L.heads, Hq = L.heads * G;
  uint4* lut = (uint4*)smem;  // [16]
  init_lut(lut, threadIdx.x);
  uint8_t* wsm = smem + 256 + warp * kWarpSmemK;
  uint8_t* tile = wsm;
  FeedK F;
  F.init(wsm + kTile, lane);
  F.evf = ST;  // attention: the score rows stay in L2 for fused V
  __syncthreads();
  const uint32_t tile_s = smem_u32(tile);
  const uint8_t* lutb = (const uint8_t*)lut;
  // STS offsets: lane l's pack i (physical 16l + i) is row-group l >> 3,
  // channel 64(l&1) + 4i + ((l>>1)&3); even/odd i differ in bit 2 of the chunk
  const uint32_t R0 = 128u * (lane >> 3) + 64u * (lane & 1) + ((lane >> 1) & 3);
  const uint32_t X = 4u * (lane & 1);
  const uint32_t st_even = 16u * ((R0 & ~7u) | ((R0 & 7u) ^ X));
  const uint32_t st_odd = 16u * ((R0 & ~7u) | (((R0 & 7u) | 4u) ^ X));
  const int64_t nwarps = int64_t(gridDim.x) * kWK, wid = int64_t(blockIdx.x) * kWK + warp;
#if PKV_KRR  // experiment: CTA ranges dealt round-robin to the warps (non-ST only)
  const Range crg = warp_range(total, blockIdx.x, int64_t(gridDim.x));
  Range rg;
  rg.b0 = crg.b0 + warp;
  rg.b1 = crg.b1;
  const int nk = rg.b1 > rg.b0 ? int((rg.b1 - rg.b0 + kWK - 1) / kWK) : 0;
  F.stride = kWK;
  constexpr int kStepK = kWK;
#else
  const Range rg = warp_range(total, wid, nwarps);
  const int nk = int(rg.b1 - rg.b0);
  constexpr int kStepK = 1;
#endif
#if PKV_Q2
  QFrag2<NU> Q;
#else
  QFrag<NU> Q;
#endif
  int cur_u = -1;
  float* sbase = scores;
  float kmx0 = -INFINITY, kmx1 = -INFINITY;  // running max of this lane's scores (heads tq, tq + 4)
  // the unit's score maxima of this warp -> kmax[u][slot][g] (lanes with gi = 0 write)
  auto flush_max = [&](int u) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      kmx0 = fmaxf(kmx0, __shfl_xor_sync(PKV_FULL, kmx0, o));
      kmx1 = fmaxf(kmx1, __shfl_xor_sync(PKV_FULL, kmx1, o));
    }
    const int64_t slot = wid - warp_of(int64_t(u) * NB, total, nwarps);
    float* km = kmax + (int64_t(u) * kslots + slot) * G;
    if (gi == 0 && tq < G) km[tq] = kmx0;
    if (gi == 0 && tq + 4 < G) km[tq + 4] = kmx1;
    kmx0 = kmx1 = -INFINITY;
  };
  Cursor cs;
  cs.init(rg.b0, NB, L.heads);
#if PKV_DIAG_WAITCLK
  long long dwait = 0;
  const long long tstart = clock64();
#endif
  // PDL: only the shared-memory prologue overlaps the previous kernel (which
  // may be the compressor writing the tables and arena this launch reads)
  pdl_wait();
  pdl_launch();
  F.refill(L, 0, NB, rg, nk, -1, 0u, lane);

#pragma unroll 1
  for (int k = 0; k < nk; ++k, cs.step(kStepK, NB, L.heads)) {
    const int u = cs.u, j = cs.j;
    if (u != cur_u) {
      if (ST && cur_u >= 0) flush_max(cur_u);
      cur_u = u;
      const int b = cs.b, h = cs.h;
      sbase = scores + (int64_t(b) * Hq + int64_t(h) * G) * sstride;
      build_qfrag<NU>(q + (int64_t(b) * Hq + int64_t(h) * G) * kD, G, lane, Q);
    }
    const uint8_t* gblk;
#if PKV_DIAG_WAITCLK
    const long long tw0 = clock64();
#endif
    bool have;
    const uint32_t blk = F.wait(k, &gblk, &have);
#if PKV_DIAG_WAITCLK
    dwait += clock64() - tw0;
#endif
#if PKV_DIAG_FEEDONLY
    if (have && lane == 0) sbase[j] = __uint_as_float(ld32(blk));
    if (false) {
#elif PKV_DIAG_FEEDPARSE
    if (have) {
      Chunk ch;
      const bool fast = gblk == nullptr && parse_chunk(blk, lane, lane, ch);
      if (lane == 0) sbase[j] = __uint_as_float(ch.bit + fast + ch.mn[3] + ch.nb.y);
    }
    if (false) {
#else
    if (have) {
#endif
      Chunk ch;
      // the fast path on the staged copy, or in place (global loads) on a block
      // too large for the ring
      auto fast_block = [&](auto bp) {
        // packs in pairs (two independent decode chains), loads one pair ahead
  #if PKV_DIAG_NOSTS
          uint32_t dsum = 0;
  #endif
          // the narrow-only loop unless the block holds a pack of width 5..8
          auto decode_packs = [&](auto wide) {
            uint32_t bit = ch.bit + abase(bp);
            const auto db = dbase(bp);
            uint32_t wa = w16_of(ch.nb, 0), wb = w16_of(ch.nb, 1);
            PackLd A = pack_load<PKV_KREGC>(db, lutb, bit, wa), B = pack_load<PKV_KREGC>(db, lutb, bit + wa, wb);
    #pragma unroll
            for (int i2 = 0; i2 < 16; i2 += 2) {
              const uint32_t bitA = bit, bitB = bit + wa;
              const uint32_t nbit = bitB + wb;
              uint32_t nwa = 0, nwb = 0;
              PackLd nA, nB;
              if (i2 < 14) {
                nwa = w16_of(ch.nb, i2 + 2);
                nwb = w16_of(ch.nb, i2 + 3);
                nA = pack_load<PKV_KREGC>(db, lutb, nbit, nwa);
                nB = pack_load<PKV_KREGC>(db, lutb, nbit + nwa, nwb);
              }
              uint32_t ra[4], rb[4];
    #if PKV_DIAG_NODECODE
              ra[0] = A.w0 ^ bitA; ra[1] = A.w1; ra[2] = A.w2; ra[3] = A.c.x;
              rb[0] = B.w0 ^ bitB; rb[1] = B.w1; rb[2] = B.w2; rb[3] = B.c.x;
    #else
              pack_decode<decltype(wide)::value>(db, A, bitA, wa, min_rep(ch.mn, i2), ra);
              pack_decode<decltype(wide)::value>(db, B, bitB, wb, min_rep(ch.mn, i2 + 1), rb);
    #endif
    #if PKV_DIAG_NOSTS
              dsum ^= ra[0] ^ ra[1] ^ ra[2] ^ ra[3] ^ rb[0] ^ rb[1] ^ rb[2] ^ rb[3];
    #else
              *(uint4*)(tile + st_even + 128u * (i2 >> 1)) = make_uint4(ra[0], ra[1], ra[2], ra[3]);
              *(uint4*)(tile + st_odd + 128u * (i2 >> 1)) = make_uint4(rb[0], rb[1], rb[2], rb[3]);
    #endif
              bit = nbit;
              wa = nwa;
              wb = nwb;
              if (i2 < 14) {
                A = nA;
                B = nB;
              }
            }
          };
          if (ch.wide) decode_packs(std::true_type{});
          else decode_packs(std::false_type{});
          // (scale, zp) of the rows this lane finalises: 16g + tok(gi) (+8)
          uint32_t prm[4][2];
  #pragma unroll
          for (int g = 0; g < 4; ++g) {
            prm[g][0] = ld32(bp + kPar + 4 * (16 * g + tok(gi)));
            prm[g][1] = ld32(bp + kPar + 4 * (16 * g + tok(gi) + 8));
          }
          __syncwarp();
          float* p0 = sbase + int64_t(tq) * sstride + j * kRows + tok(gi);  // rows 16g + tok(gi) (+8) of head tq
          float* p1 = p0 + 4 * sstride;                                     // head tq + 4
  #if PKV_DIAG_NOMMA
  #if PKV_DIAG_NOSTS
          if (tq < G) p0[0] = __uint_as_float(dsum) + __uint_as_float(prm[0][0]);
  #else
          if (tq < G) p0[0] = __uint_as_float(ld32(tile_s + 16u * lane)) + __uint_as_float(prm[0][0]);
  #endif
  #else
  #pragma unroll
          for (int g = 0; g < 4; ++g) {
            int accU[NU][4], accS[4];
  #pragma unroll
            for (int e = 0; e < 4; ++e) {
              accS[e] = 0;
  #pragma unroll
              for (int nu = 0; nu < NU; ++nu) accU[nu][e] = 0;
            }
            // lane L addresses row R = 128g + 32jj + L
            const uint32_t a0 = tile_s + 16u * (128u * g + lane);              // jj = 0, 1 (+512 B)
            const uint32_t a1 = tile_s + 16u * (128u * g + (lane ^ 4u) + 64u);  // jj = 2, 3
  #pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              uint32_t a[4];
              ldsm_t(a, (jj < 2 ? a0 : a1) + 512u * (jj & 1));
                k_mma<NU>(accU, accS, a, Q, jj);
            }
            const float sA = h2f(prm[g][0] & 0xffff), zA = h2f(prm[g][0] >> 16);
            const float sB = h2f(prm[g][1] & 0xffff), zB = h2f(prm[g][1] >> 16);
            // digit sums: d0 + 256*d1 <= 128*255*65535 < 2^31 is exact in int32
            if (tq < G) {
              const float vA = k_val<NU>(accU, accS, Q, 0, 0);
              const float vB = k_val<NU>(accU, accS, Q, 0, 1);
              const float scA = fmaf(sA, vA * Q.inv[0], zA * Q.qs[0]), scB = fmaf(sB, vB * Q.inv[0], zB * Q.qs[0]);
              p0[16 * g] = scA;
              p0[16 * g + 8] = scB;
              if (ST) kmx0 = fmaxf(kmx0, fmaxf(scA, scB));
            }
            if (NU == 2 && tq + 4 < G) {
              const float vA = k_val<NU>(accU, accS, Q, NU - 1, 0);
              const float vB = k_val<NU>(accU, accS, Q, NU - 1, 1);
              const float scA = fmaf(sA, vA * Q.inv[1], zA * Q.qs[1]), scB = fmaf(sB, vB * Q.inv[1], zB * Q.qs[1]);
              p1[16 * g] = scA;
              p1[16 * g + 8] = scB;
              if (ST) kmx1 = fmaxf(kmx1, fmaxf(scA, scB));
            }
          }
  #endif
          __syncwarp();  // tile reads done before the next block's stores
      };
      bool fast;
      if (gblk == nullptr) {
        fast = parse_chunk(blk, lane, lane, ch);
        if (fast) fast_block(blk);
      } else {
        fast = parse_chunk(gblk, lane, lane, ch);
        if (fast) fast_block(gblk);
      }
      if (!fast) {
        // scalar path (rare): lane computes rows lane and lane+32 for every head
        const int b = u / L.heads, h = u - b * L.heads;
        const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * kD;
        float* srow = sbase + j * kRows;
        uint32_t* desc = (uint32_t*)tile;
        const uint8_t* bg = gblk ? gblk : gptr(blk);
        if (gblk) parse_chunk(bg, lane, lane, ch);
        build_desc(ch, lane, desc);
#pragma unroll 1
        for (int half = 0; half < 2; ++half) {
          const int tt = lane + 32 * half, rgp = tt >> 4, t16 = tt & 15;
          const uint32_t pr = ld32(bg + kPar + 4 * tt);
          const float s = h2f(pr & 0xffff), z = h2f(pr >> 16);
#pragma unroll 1
          for (int g = 0; g < G; ++g) {
            float acc = 0.f, qsum = 0.f;
#pragma unroll 1
            for (int pos = 0; pos < 128; ++pos) {
              const uint32_t d = desc[rgp * 128 + pos];
              const uint32_t wd = d >> 18;
              const float code = float(pack_min(bg, rgp * 128 + pos) + field_at(bg, (d & 0x3ffffu) + t16 * wd, wd));
              const float qc = qu[g * kD + kpos_to_col(pos, kD)];
              acc = fmaf(code, qc, acc);
              qsum += qc;
            }
            const float sc = fmaf(s, acc, z * qsum);
            srow[int64_t(g) * sstride + tt] = sc;
            if (ST) {  // fold into the lanes that own head g's running max
              const float m = warp_max(sc);
              if ((g & 3) == tq) {
                if (g < 4) kmx0 = fmaxf(kmx0, m);
                else kmx1 = fmaxf(kmx1, m);
              }
            }
          }
        }
        __syncwarp();
      }
    }
    F.refill(L, 0, NB, rg, nk, k, F.tail_after(k), lane);
  }
  if (ST && cur_u >= 0) flush_max(cur_u);
#if PKV_DIAG_WAITCLK
  __syncwarp();
  if (lane == 0) {  // (wait cycles, loop cycles, blocks) per warp at the start of scores
    long long* dbg = reinterpret_cast<long long*>(scores) + 3 * wid;
    dbg[0] = dwait;
    dbg[1] = clock64() - tstart;
    dbg[2] = nk;
  }
  return;
#endif
  // uncompressed residue rows (< 64 per sequence): unit u = wid, wid + nwarps,
  // ... on one warp, lane per token (independent dot products, no shuffle
  // chains), the unit's q staged in the warp's tile
  for (int64_t uu = wid; uu < U; uu += nwarps) {
    const int u = int(uu);
    const int b = u / L.heads, h = u - b * L.heads;
    const int nr = res_rows(L, b, sstride);
    float rm[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) rm[g] = -INFINITY;
    if (nr > 0) {
      const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * kD;
      float* qs = reinterpret_cast<float*>(tile);
      __syncwarp();
      for (int i = lane; i < G * kD / 4; i += 32) reinterpret_cast<float4*>(qs)[i] = reinterpret_cast<const float4*>(qu)[i];
      __syncwarp();
      float* srow = scores + (int64_t(b) * Hq + int64_t(h) * G) * sstride + int64_t(L.nblk[b]) * kRows;
      for (int t = lane; t < nr; t += 32) {
        const uint4* kr = reinterpret_cast<const uint4*>(L.stage + (int64_t(u) * L.buffer + t) * kD);
        float acc[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) acc[g] = 0.f;
#pragma unroll 4
        for (int c8 = 0; c8 < kD / 8; ++c8) {
          const uint4 v = kr[c8];
          const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float x0 = h2f(wv[e] & 0xffff), x1 = h2f(wv[e] >> 16);
#pragma unroll
            for (int g = 0; g < 8; ++g)
              if (g < G) {
                const float2 qv = *reinterpret_cast<const float2*>(qs + g * kD + 8 * c8 + 2 * e);
                acc[g] = fmaf(x1, qv.y, fmaf(x0, qv.x, acc[g]));
              }
          }
        }
#pragma unroll
        for (int g = 0; g < 8; ++g)
          if (g < G) {
            srow[int64_t(g) * sstride + t] = acc[g];
            rm[g] = fmaxf(rm[g], acc[g]);
          }
      }
    }
    if (ST) {
#pragma unroll
      for (int g = 0; g < 8; ++g)
        if (g < G) {
          const float m = warp_max(rm[g]);
          if (lane == 0) kres[int64_t(u) * G + g] = m;
        }
    }
  }
}

// ======================================================================= V
// Lane (gi, tq) decodes physical packs 128tq + 16gi + i (row-group tq, channel
// 16gi + i), i = 0..15, two per m-tile: rows gi / gi+8 of m-tile mt are
// channels 16gi + 2mt / +1.  k-chunk tq <-> row-group tq bytes 0..3 (k-step 0)
// / 8..11 (k-step 1), chunk tq+4 <-> bytes 4..7 / 12..15.  The B operand
// (rows x [head, digit]) comes from a per-warp [head][digit][64] byte array
// in the same byte order.  D columns 2tq, 2tq+1 = head tq digits 0, 1, so lane
// (gi, tq) owns out[head 4nt + tq][channels 16gi .. 16gi+15].  Per (warp,
// range segment = unit) partial sums go to scratch; the finalize kernel adds
// them in a fixed order (deterministic) plus the residue.
constexpr int kPart = kD + 4;  // 128 channels, the z term, l (attention), padding (16-byte rows)

// Row maximum of head g of unit u over the K launch's warp slots and residue
// rows; the `nl` lanes of a group share the loads and reduce with shuffles.
__device__ __forceinline__ float row_max(const float* __restrict__ kmax, const float* __restrict__ kres, int u, int g,
                                         int G, int NB, int64_t ktotal, int64_t knwarps, int kslots, int sub, int nl) {
  float m = sub == 0 ? kres[int64_t(u) * G + g] : -INFINITY;
  if (ktotal > 0) {
    const int64_t w0 = warp_of(int64_t(u) * NB, ktotal, knwarps), w1 = warp_of(int64_t(u + 1) * NB - 1, ktotal, knwarps);
    for (int64_t sl = sub; sl <= w1 - w0; sl += nl) m = fmaxf(m, kmax[(int64_t(u) * kslots + sl) * G + g]);
  }
  for (int o = 1; o < nl; o <<= 1) m = fmaxf(m, __shfl_xor_sync(PKV_FULL, m, o));
  return m;
}
constexpr int kWV = 4;
#ifndef PKV_VPIPE  // V: load the next pack pair while decoding the current one
#define PKV_VPIPE 1
#endif
#ifndef PKV_VMINB  // V: CTAs per SM the register allocation must allow
#define PKV_VMINB 4
#endif
#ifndef PKV_VMINB2  // the same for the G <= 8 instantiation (two n-tiles: 168 registers, no spills; config E V 624 -> 514 us)
#define PKV_VMINB2 3
#endif
#ifndef PKV_RBV  // V ring: 11 KB still fits 4 register-bound CTAs per SM (measured ~2% over 10 KB)
#define PKV_RBV 11264
#endif
constexpr int kRBV = PKV_RBV, kNSV = 3;
using FeedV = Feed<kRBV, kNSV>;
constexpr size_t kWarpSmemV = (2048 + FeedV::bytes() + 127) / 128 * 128;

// SM (attention_decode): `w` holds raw (scaled) scores instead of softmax
// weights; every block uses p_t = exp(s_t - M) with M the row maximum from
// the K launch's statistics (kmax over its kslots warp slots, kres), so no
// rescaling is ever needed, and each partial slot also carries l = sum p.
template <int NT, bool SM>  // NT: n-tiles, 1 for G <= 4, 2 for G <= 8
__global__ void __launch_bounds__(kWV * 32, NT == 2 ? PKV_VMINB2 : PKV_VMINB) fused_v_fast_kernel(pkv_layer_t L, const float* __restrict__ w, int G,
                                                                 int64_t wstride, float* __restrict__ part, int NB,
                                                                 int64_t total, int maxseg,
                                                                 float* __restrict__ vscr,
                                                                 const float* __restrict__ kmax,
                                                                 const float* __restrict__ kres, int kslots,
                                                                 int64_t knwarps, int64_t ktotal) {
  constexpr int GP = 4 * NT;    // padded heads
  constexpr int LPH = 32 / GP;  // writer lanes per head
  constexpr int TPL = 64 / LPH; // rows per writer lane (8 or 16)
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int Hq = L.heads * G;
  uint4* lut = (uint4*)smem;  // [16]
  init_lut(lut, threadIdx.x);
  uint8_t* wsm = smem + 256 + warp * kWarpSmemV;
  // 2 KB: the B operand staging [GP][2][64] (<= 1 KB), reused as the slow
  // path's descriptor table [512] after the B fragments are in registers
  uint32_t* desc = (uint32_t*)wsm;
  uint8_t* frag = wsm;
  FeedV F;
  F.init(wsm + 2048, lane);
  F.evf = SM;  // attention: the partials stay in L2 for the finalize
  __syncthreads();
  const uint8_t* lutb = (const uint8_t*)lut;
  const int64_t nwarps = int64_t(gridDim.x) * kWV, wid = int64_t(blockIdx.x) * kWV + warp;
  float* vsl = vscr + wid * (8 * kD);  // scalar-path partials [8][kD]
  // writer role for the B operand: head wh, rows wt0 .. wt0 + TPL - 1
  const int wh = lane / LPH, wt0 = (lane % LPH) * TPL;
  // Work split.  G <= 4: one contiguous, equal-length range per warp.  G <= 8
  // (RR): CTA c owns the contiguous range [total c / C, total (c+1) / C), dealt
  // round-robin to its kWV warps (warp w takes blocks w, w + kWV, ...), so the
  // warps of a CTA decode the same mix of heads; measured config E attention
  // 1105 -> 1020 us, while config B's V ran ~2% slower with it.  Partial slots
  // are per (unit, warp) or per (unit, CTA, warp); a warp writes zeros for the
  // units of its range it gets no block of.
  constexpr bool RR = NT == 2;
  const int64_t ncta = gridDim.x;
  const Range crg = RR ? warp_range(total, blockIdx.x, ncta) : warp_range(total, wid, nwarps);
  Range rg;
  rg.b0 = RR ? crg.b0 + warp : crg.b0;
  rg.b1 = crg.b1;
  constexpr int kStep = RR ? kWV : 1;
  const int nk = rg.b1 > rg.b0 ? int((rg.b1 - rg.b0 + kStep - 1) / kStep) : 0;
  F.stride = kStep;
  const int u_first = int(crg.b0 / NB);
  const int u_last = crg.b1 > crg.b0 ? int((crg.b1 - 1) / NB) : u_first - 1;

  float acc[NT][16];
  float zacc = 0.f, lacc = 0.f;
  float Mh = 0.f;  // SM: row maximum (times log2 e) of the writer head wh for the current unit
  bool slow_used = false;
  int seg = 0;  // segment (unit - u_first) the accumulators belong to
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[nt][i] = 0.f;
  // write the accumulators of segment `seg` (then zero them)
  auto flush = [&]() {
    // partials of unit u go to slot (this warp - first warp covering u), or
    // (RR) (this CTA - first CTA covering u) * kWV + warp
    const int u = u_first + seg;
    const int64_t slot = RR ? (int64_t(blockIdx.x) - warp_of(int64_t(u) * NB, total, ncta)) * kWV + warp
                            : wid - warp_of(int64_t(u) * NB, total, nwarps);
    float* pp = part + (int64_t(u) * maxseg + slot) * G * kPart;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int g = 4 * nt + tq;
      if (g < G) {
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4)
          *(float4*)(pp + g * kPart + 16 * gi + 4 * i4) =
              make_float4(acc[nt][4 * i4], acc[nt][4 * i4 + 1], acc[nt][4 * i4 + 2], acc[nt][4 * i4 + 3]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[nt][i] = 0.f;
    }
    float z = zacc, l = lacc;
#pragma unroll
    for (int o = 1; o < LPH; o <<= 1) {
      z += __shfl_xor_sync(PKV_FULL, z, o);
      if (SM) l += __shfl_xor_sync(PKV_FULL, l, o);
    }
    if (lane % LPH == 0 && wh < G) {
      pp[wh * kPart + kD] = z;
      if (SM) pp[wh * kPart + kD + 1] = l;
    }
    zacc = lacc = 0.f;
    if (slow_used) {
      __syncwarp();
      for (int e = lane; e < G * kD; e += 32) {
        const int g = e / kD, c = e - g * kD;
        pp[g * kPart + c] += vsl[g * kD + c];
        vsl[g * kD + c] = 0.f;
      }
      slow_used = false;
    }
    ++seg;
  };

  // weights of the next block (prefetched one block ahead); vector loads when
  // every row starts 16-byte aligned, else scalar (any w_stride)
  const bool wvec = (wstride & 3) == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0;
  float wn[TPL];
  auto load_w = [&](int k, const Cursor& c) {
    const float* wrow = w + (int64_t(c.b) * Hq + int64_t(c.h) * G + wh) * wstride + int64_t(c.j) * kRows + wt0;
    const bool ok = k < nk && wh < G;
#pragma unroll
    for (int q4 = 0; q4 < TPL / 4; ++q4) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ok) {
        if (wvec) {
          v = *(const float4*)(wrow + 4 * q4);
        } else {  // any row stride (rows not 16-byte aligned): scalar loads
          v.x = wrow[4 * q4]; v.y = wrow[4 * q4 + 1]; v.z = wrow[4 * q4 + 2]; v.w = wrow[4 * q4 + 3];
        }
      }
      wn[4 * q4] = v.x; wn[4 * q4 + 1] = v.y; wn[4 * q4 + 2] = v.z; wn[4 * q4 + 3] = v.w;
    }
  };
  Cursor cs, cn;
  cs.init(rg.b0, NB, L.heads);
  cn = cs;
  int cur_u = -1, b = 0, h = 0;
#if PKV_DIAG_WAITCLK
  long long dwait = 0;
  const long long tstart = clock64();
#endif
  // PDL: only the shared-memory prologue overlaps the previous kernel (the K
  // launch writing the scores, or a compressor writing the tables)
  pdl_wait();
  pdl_launch();
  F.refill(L, 1, NB, rg, nk, -1, 0u, lane);
  load_w(0, cn);

#pragma unroll 1
  for (int k = 0; k < nk; ++k) {
    const int u = cs.u, j = cs.j;
    if (u != cur_u) {
      cur_u = u;
      b = cs.b;
      h = cs.h;
      if (SM) Mh = row_max(kmax, kres, u, wh < G ? wh : 0, G, NB, ktotal, knwarps, kslots, lane % LPH, LPH) * 1.4426950408889634f;
    }
    while (seg < u - u_first) flush();
    float wc[TPL];
#pragma unroll
    for (int e = 0; e < TPL; ++e) wc[e] = wn[e];
    cn.step(kStep, NB, L.heads);
    load_w(k + 1, cn);
    cs = cn;
    const uint8_t* gblk;
#if PKV_DIAG_WAITCLK
    const long long tw0 = clock64();
#endif
    bool have;
    const uint32_t sblk = F.wait(k, &gblk, &have);
#if PKV_DIAG_WAITCLK
    dwait += clock64() - tw0;
#endif
    // one block: B operand, then the IMMA fast path or the scalar path.  Called
    // with the shared-memory copy (LDS), or for a block too large to stage with
    // the global-memory block (generic loads, scalar path only).
    auto process = [&](auto blk, bool may_fast) {
      Chunk ch;
      const int src = 8 * tq + gi;  // the chunk this lane decodes (row-group tq, channels 16gi..)
      // ---- B operand: x_t = w_t * s_t as 2 unsigned byte digits scaled per
      // (block, head) by f = 65535 / max x, so every x is rounded to nearest at
      // 2^-16 of the block's largest (the digit sums are exact in int32); z term
      // sum_t w_t z_t in f32.  A block with a negative x (w is any real vector,
      // SPEC.md:455-463; softmax weights never are) takes the scalar f32 path:
      // signed digits would lose the precision the code / zero-point cancellation
      // needs (out = sum x*code + sum w*z nearly cancels on centred V).
      // The parse (loads, flags, scan) and the operand (params, x, max) are
      // independent chains: loads first, one vote, the two shuffle chains
      // interleaved.
      parse_load(blk, lane, src, ch);
      uint2 pr[TPL / 2];
#pragma unroll
      for (int e2 = 0; e2 < TPL / 2; ++e2) pr[e2] = ld64(blk + kPar + 4 * (wt0 + 2 * e2));
      float xs[TPL];
      float mx = 0.f;
      bool neg = false;
      if (SM) {
#pragma unroll
        for (int e = 0; e < TPL; ++e) {
          wc[e] = exp2f(fmaf(wc[e], 1.4426950408889634f, -Mh));  // p_t = exp(s_t - M)
          lacc += wc[e];
        }
      }
#pragma unroll
      for (int e2 = 0; e2 < TPL / 2; ++e2) {
        const float s0 = h2f(pr[e2].x & 0xffff), s1 = h2f(pr[e2].y & 0xffff);
        zacc = fmaf(wc[2 * e2], h2f(pr[e2].x >> 16), fmaf(wc[2 * e2 + 1], h2f(pr[e2].y >> 16), zacc));
        xs[2 * e2] = wc[2 * e2] * s0;
        xs[2 * e2 + 1] = wc[2 * e2 + 1] * s1;
        mx = fmaxf(mx, fmaxf(xs[2 * e2], xs[2 * e2 + 1]));
        neg |= (xs[2 * e2] < 0.f) | (xs[2 * e2 + 1] < 0.f);
      }
      const uint32_t flags = parse_flags(ch) | (neg ? uint32_t(kFNeg) : 0u);
      const bool fast = parse_verdict(__reduce_or_sync(PKV_FULL, flags), ch) && may_fast;
      parse_scan(lane, ch);
#pragma unroll
      for (int o = 1; o < LPH; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(PKV_FULL, mx, o));
      // (f only needs f * invf ~ 1 and max x * f <= 65535.5, the clamp below)
      const float f = mx > 1e-30f ? __fdividef(65535.f, mx) : 0.f;
      const float invf = mx * (1.f / 65535.f);
#pragma unroll
      for (int e8 = 0; e8 < TPL / 8; ++e8) {
        uint32_t v[8];
#pragma unroll
        // round to nearest (unbiased: a softmax-weighted block sums many small
        // x·f with errors of both signs), clamped so 65535.5+ cannot carry
        for (int e = 0; e < 8; ++e) v[e] = min(__float_as_uint(__fmaf_rn(xs[8 * e8 + e], f, 8388608.f)), 0x4B00FFFFu);
        const uint32_t t01 = __byte_perm(v[0], v[1], 0x5140), t45 = __byte_perm(v[4], v[5], 0x5140);
        const uint32_t t23 = __byte_perm(v[2], v[3], 0x5140), t67 = __byte_perm(v[6], v[7], 0x5140);
        const uint32_t lo0 = __byte_perm(t01, t45, 0x5410), hi0 = __byte_perm(t01, t45, 0x7632);
        const uint32_t lo1 = __byte_perm(t23, t67, 0x5410), hi1 = __byte_perm(t23, t67, 0x7632);
        *(uint2*)(frag + (wh * 2 + 0) * 64 + wt0 + 8 * e8) = make_uint2(lo0, lo1);
        *(uint2*)(frag + (wh * 2 + 1) * 64 + wt0 + 8 * e8) = make_uint2(hi0, hi1);
      }
      __syncwarp();
      uint32_t bf[NT][4];
      float inv[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const uint4 v = *(const uint4*)(frag + ((4 * nt + (gi >> 1)) * 2 + (gi & 1)) * 64 + 16 * tq);
        bf[nt][0] = v.x; bf[nt][1] = v.y; bf[nt][2] = v.z; bf[nt][3] = v.w;
        inv[nt] = __shfl_sync(PKV_FULL, invf, (4 * nt + tq) * LPH);
      }
      __syncwarp();  // frag reads done (the slow path reuses the area)
      if (fast) {
        // lane (gi, tq) = chunk 8tq + gi of the scan (its minima are in ch.mn)
        uint32_t bit = __shfl_sync(PKV_FULL, ch.bit, src) + abase(blk);
        const auto db = dbase(blk);
        const uint2 nb = ld64(blk + kNib + 8 * src);
        const uint32_t (&mn)[8] = ch.mn;
        // the m-tile's two packs decoded together, the next pair's loads in flight
        auto decode_mma = [&](auto wide) {
#if PKV_VPIPE
          uint32_t wa = w16_of(nb, 0), wb = w16_of(nb, 1);
          PackLd A = pack_load(db, lutb, bit, wa), B = pack_load(db, lutb, bit + wa, wb);
#endif
  #pragma unroll
          for (int mt = 0; mt < 8; ++mt) {
            uint32_t P[2][4];
#if !PKV_VPIPE
            {  // no cross-pair load pipelining: fewer live registers, latency hidden by more warps
              const int i2 = 2 * mt;
              const uint32_t wa = w16_of(nb, i2), wb = w16_of(nb, i2 + 1);
              const PackLd A = pack_load(db, lutb, bit, wa), B = pack_load(db, lutb, bit + wa, wb);
              pack_decode<decltype(wide)::value>(db, A, bit, wa, min_rep(mn, i2), P[0]);
              pack_decode<decltype(wide)::value>(db, B, bit + wa, wb, min_rep(mn, i2 + 1), P[1]);
              bit += wa + wb;
            }
#else
            {
              const int i2 = 2 * mt;
              const uint32_t bitA = bit, bitB = bit + wa;
              const uint32_t nbit = bitB + wb;
              uint32_t nwa = 0, nwb = 0;
              PackLd nA, nB;
              if (i2 < 14) {
                nwa = w16_of(nb, i2 + 2);
                nwb = w16_of(nb, i2 + 3);
                nA = pack_load(db, lutb, nbit, nwa);
                nB = pack_load(db, lutb, nbit + nwa, nwb);
              }
              pack_decode<decltype(wide)::value>(db, A, bitA, wa, min_rep(mn, i2), P[0]);
              pack_decode<decltype(wide)::value>(db, B, bitB, wb, min_rep(mn, i2 + 1), P[1]);
              bit = nbit;
              wa = nwa;
              wb = nwb;
              if (i2 < 14) {
                A = nA;
                B = nB;
              }
            }
#endif
  #pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              int d[4] = {0, 0, 0, 0};
              const uint32_t a0[4] = {P[0][0], P[1][0], P[0][1], P[1][1]};
              imma_uu(d, a0, bf[nt][0], bf[nt][1]);
              const uint32_t a1[4] = {P[0][2], P[1][2], P[0][3], P[1][3]};
              imma_uu(d, a1, bf[nt][2], bf[nt][3]);
              acc[nt][2 * mt] = fmaf(float(d[0] + 256 * d[1]), inv[nt], acc[nt][2 * mt]);
              acc[nt][2 * mt + 1] = fmaf(float(d[2] + 256 * d[3]), inv[nt], acc[nt][2 * mt + 1]);
            }
          }
        };
        if (ch.wide) decode_mma(std::true_type{});
        else decode_mma(std::false_type{});
      } else {
        // scalar path (rare): lane owns channels lane + 32q, all 64 rows, all heads;
        // partials accumulate in this warp's global scratch (fixed order, deterministic)
        build_desc(ch, lane, desc);
        if (!slow_used) {
          for (int e = lane; e < 8 * kD; e += 32) vsl[e] = 0.f;
          __syncwarp();
          slow_used = true;
        }
        const float* wu = w + (int64_t(b) * Hq + int64_t(h) * G) * wstride + int64_t(j) * kRows;
        float Mg[8];  // SM: every head's row maximum (from its writer lanes)
#pragma unroll
        for (int g = 0; g < 8; ++g) Mg[g] = __shfl_sync(PKV_FULL, Mh, (g < GP ? g : 0) * LPH);
        float sacc[8][4];
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) sacc[g][q4] = vsl[g * kD + lane + 32 * q4];
#pragma unroll 1
        for (int r = 0; r < kRows; ++r) {
          const uint32_t pr = ld32(gptr(blk) + kPar + 4 * r);
          const float s = h2f(pr & 0xffff);
          float ws[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) {
          float wv = g < G ? wu[int64_t(g) * wstride + r] : 0.f;
          if (SM && g < G) wv = exp2f(fmaf(wv, 1.4426950408889634f, -Mg[g]));
          ws[g] = wv * s;
        }
          const int rgp = r >> 4, tt = r & 15;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int c = lane + 32 * q4;
            const uint32_t dd = desc[rgp * 128 + c];
            const uint32_t wd = dd >> 18;
            const float code = float(pack_min(gptr(blk), rgp * 128 + c) + field_at(gptr(blk), (dd & 0x3ffffu) + tt * wd, wd));
#pragma unroll
            for (int g = 0; g < 8; ++g) sacc[g][q4] = fmaf(ws[g], code, sacc[g][q4]);
          }
        }
#pragma unroll
        for (int g = 0; g < 8; ++g)
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) vsl[g * kD + lane + 32 * q4] = sacc[g][q4];
      }
      __syncwarp();
    };
    if (have) {
      if (gblk)
        process(gblk, false);
      else
        process(sblk, true);  // the shared-window address (LDS, 32-bit addressing)
    }
    F.refill(L, 1, NB, rg, nk, k, F.tail_after(k), lane);
  }
#if PKV_DIAG_WAITCLK
  __syncwarp();
  if (lane == 0) {  // (wait cycles, loop cycles, blocks) per warp at the start of the partials
    long long* dbg = reinterpret_cast<long long*>(part) + 3 * wid;
    dbg[0] = dwait;
    dbg[1] = clock64() - tstart;
    unsigned smid;  // blocks | SM id << 32 (tools/exp/waitclk_v.py)
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    dbg[2] = nk | (int64_t(smid) << 32);
  }
  return;
#endif
  while (seg <= u_last - u_first) flush();
}

// out[b][h*G+g][c] = sum over the warps whose range meets unit u (ascending) of
// their partials (channels and z term), plus the residue rows.  One CTA of 512
// threads per (unit, head): thread (q, c) sums slots q, q+4, ... of channel c
// (eight loads in flight), then the four quarter sums are added in a fixed
// order (deterministic).  SM: `w` holds scores; the result is divided by the
// softmax denominator (sum of the slots' l plus the residue rows' weights).
template <bool SM>
__global__ void __launch_bounds__(512) fused_v_fast_finalize(pkv_layer_t L, const float* __restrict__ part,
                                                              const float* __restrict__ w, int G, int64_t wstride,
                                                              int NB, int64_t total, int64_t nranges, int spc,
                                                              int maxseg,
                                                              float* __restrict__ out, const float* __restrict__ kmax,
                                                              const float* __restrict__ kres, int kslots,
                                                              int64_t knwarps, int64_t ktotal) {
  __shared__ float red[4][kD + 2];
  __shared__ float Msh;
  const int U = L.batch * L.heads;
  const int c = threadIdx.x & 127, qq = threadIdx.x >> 7;
  pdl_wait();  // the V partials
  pdl_launch();
  for (int ug = blockIdx.x; ug < U * G; ug += gridDim.x) {
    const int u = ug / G, g = ug - u * G;
    if (SM && threadIdx.x < 32) {
      const float m = row_max(kmax, kres, u, g, G, NB, ktotal, knwarps, kslots, threadIdx.x, 32);
      if (threadIdx.x == 0) Msh = m;
    }
    float s = 0.f, z = 0.f, l = 0.f;
    if (total > 0 && NB > 0) {
      // slots: spc per range meeting the unit (fused_v_fast_kernel: 1 per warp range, kWV per CTA range)
      const int64_t w0 = warp_of(int64_t(u) * NB, total, nranges), w1 = warp_of(int64_t(u + 1) * NB - 1, total, nranges);
      const int ns = int(w1 - w0 + 1) * spc;
      const float* pp = part + (int64_t(u) * maxseg * G + g) * kPart;
      const int64_t st = int64_t(G) * kPart;
      // eight independent partial sums (loads in flight), combined in a fixed order
      float a[8], bz[8], bl[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = bz[i] = bl[i] = 0.f;
      int sl = qq;
      for (; sl + 28 < ns; sl += 32) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          a[i] += pp[(sl + 4 * i) * st + c];
          bz[i] += pp[(sl + 4 * i) * st + kD];
          if (SM) bl[i] += pp[(sl + 4 * i) * st + kD + 1];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (sl + 4 * i < ns) {
          a[i] += pp[(sl + 4 * i) * st + c];
          bz[i] += pp[(sl + 4 * i) * st + kD];
          if (SM) bl[i] += pp[(sl + 4 * i) * st + kD + 1];
        }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s += a[i];
        z += bz[i];
        l += bl[i];
      }
    }
    // residue rows (< 64): row t goes to thread group t % 4, 8 loads in flight
    {
      const int b = u / L.heads;
      const int nr = res_rows(L, b, wstride);
      const float* wr = w + (int64_t(b) * L.heads * G + int64_t(u - b * L.heads) * G + g) * wstride + int64_t(L.nblk[b]) * kRows;
      const uint16_t* vr = L.stage + (int64_t(1) * U + u) * L.buffer * kD;
      if (SM) __syncthreads();  // Msh
      const float M = SM ? Msh : 0.f;
      for (int t0 = qq; t0 < nr; t0 += 32) {
        float pw[8], xv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int t = t0 + 4 * i < nr ? t0 + 4 * i : t0;
          pw[i] = wr[t];
          xv[i] = __half2float(__ushort_as_half(vr[t * kD + c]));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (t0 + 4 * i < nr) {
            const float p = SM ? expf(pw[i] - M) : pw[i];
            s = fmaf(p, xv[i], s);
            l += p;
          }
      }
    }
    red[qq][c] = s;
    if (c == 0) {
      red[qq][kD] = z;
    }
    // l: every thread of a group holds the same residue sum; the slot sums sit in c == 0
    if (c == 0) red[qq][kD + 1] = l;
    __syncthreads();
    if (qq == 0) {
      s = ((red[0][c] + red[1][c]) + red[2][c]) + red[3][c];
      z = ((red[0][kD] + red[1][kD]) + red[2][kD]) + red[3][kD];
      l = ((red[0][kD + 1] + red[1][kD + 1]) + red[2][kD + 1]) + red[3][kD + 1];
      out[int64_t(ug) * kD + c] = SM ? (s + z) / l : s + z;
    }
    __syncthreads();
  }
}

constexpr size_t k_smem_bytes() { return 256 + kWK * kWarpSmemK; }
constexpr size_t v_smem_bytes() { return 256 + kWV * kWarpSmemV; }

// CTAs that fit on the device at once (queried once per kernel; the grid is
// never larger, so every warp's range is resident for the whole launch)
template <class K>
int fast_grid(K kernel, int threads, size_t smem, int64_t work_warps, int wpc) {
  // resident CTAs per device for each kernel instantiation, queried once
  // (occupancy queries cost microseconds per call); thread-safe, per device
  struct Cap {
    const void* k;
    int dev, cap;
  };
  static std::mutex mu;
  static std::vector<Cap> caps;
  int dev = 0;
  cudaGetDevice(&dev);
  int cap = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Cap& c : caps)
      if (c.k == (const void*)kernel && c.dev == dev) cap = c.cap;
  }
  if (!cap) {
    int nsm = 0, per = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
    cap = max(1, per) * nsm;
    std::lock_guard<std::mutex> lock(mu);
    caps.push_back({(const void*)kernel, dev, cap});
  }
  const int64_t want = (work_warps + wpc - 1) / wpc;
  return int(want < 1 ? 1 : (want < cap ? want : cap));
}

// grids (CTAs resident at once, never more than the work needs)
template <bool SM>
int v_grid(const pkv_layer_t* L, int nblocks, int G) {
  const int64_t total = int64_t(L->batch) * L->heads * nblocks;
  return G <= 4 ? fast_grid(fused_v_fast_kernel<1, SM>, kWV * 32, v_smem_bytes(), total, kWV)
                : fast_grid(fused_v_fast_kernel<2, SM>, kWV * 32, v_smem_bytes(), total, kWV);
}
template <bool ST>
int k_grid(const pkv_layer_t* L, int nblocks, int G) {
  const int64_t total = int64_t(L->batch) * L->heads * nblocks;
  const int64_t U = int64_t(L->batch) * L->heads;
  const int64_t ww = total > U ? total : U;  // at least one warp per unit for the residue
  return G <= 4 ? fast_grid(fused_k_fast_kernel<1, ST>, kWK * 32, k_smem_bytes(), ww, kWK)
                : fast_grid(fused_k_fast_kernel<2, ST>, kWK * 32, k_smem_bytes(), ww, kWK);
}
// slots per unit: the most warps whose ranges can meet one unit
int v_maxseg(const pkv_layer_t* L, int nblocks, int64_t nwarps) {
  const int64_t total = int64_t(L->batch) * L->heads * nblocks;
  if (nblocks <= 0 || total <= 0) return 1;
  const int64_t len_min = total / nwarps;  // every range has len_min or len_min + 1 blocks
  if (len_min == 0) return int(nblocks < nwarps ? nblocks : nwarps) + 1;
  return int((nblocks + len_min - 1) / len_min + 1);
}
// V partial slots per unit: kWV per CTA range that can meet one unit
int v_slots(const pkv_layer_t* L, int nblocks, int64_t ncta) { return kWV * v_maxseg(L, nblocks, ncta); }
int64_t v_part_floats(const pkv_layer_t* L, int maxseg, int G, int64_t nwarps) {
  return int64_t(L->batch) * L->heads * maxseg * G * kPart + nwarps * 8 * kD;
}

template <bool ST>
void launch_k(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride, float* kmax,
              float* kres, int kslots, cudaStream_t s) {
  const int64_t total = int64_t(L->batch) * L->heads * nblocks;
  const int NB = max(1, nblocks);
  const int grid = k_grid<ST>(L, nblocks, G);
  if (G <= 4)
    pkv_launch_pdl(fused_k_fast_kernel<1, ST>, grid, kWK * 32, k_smem_bytes(), s, *L, q, G, scores, sstride, NB, total,
                   kmax, kres, kslots);
  else
    pkv_launch_pdl(fused_k_fast_kernel<2, ST>, grid, kWK * 32, k_smem_bytes(), s, *L, q, G, scores, sstride, NB, total,
                   kmax, kres, kslots);
}

template <bool SM>
void launch_v(const pkv_layer_t* L, int nblocks, const float* w, int G, int64_t wstride, float* out, float* part,
              const float* kmax, const float* kres, int kslots, int64_t knwarps, cudaStream_t s) {
  const int64_t total = int64_t(L->batch) * L->heads * nblocks;
  const int grid = v_grid<SM>(L, nblocks, G);
  const int64_t nwarps = int64_t(grid) * kWV;
  const bool rr = G > 4;  // the NT = 2 instantiation deals CTA ranges round-robin
  const int maxseg = rr ? v_slots(L, nblocks, grid) : v_maxseg(L, nblocks, nwarps);
  const int NB = max(1, nblocks);
  float* vscr = part + int64_t(L->batch) * L->heads * maxseg * G * kPart;
  if (total > 0) {
    if (G <= 4)
      pkv_launch_pdl(fused_v_fast_kernel<1, SM>, grid, kWV * 32, v_smem_bytes(), s, *L, w, G, wstride, part, NB, total,
                     maxseg, vscr, kmax, kres, kslots, knwarps, total);
    else
      pkv_launch_pdl(fused_v_fast_kernel<2, SM>, grid, kWV * 32, v_smem_bytes(), s, *L, w, G, wstride, part, NB, total,
                     maxseg, vscr, kmax, kres, kslots, knwarps, total);
  }
  const int ug = L->batch * L->heads * G;
  pkv_launch_pdl(fused_v_fast_finalize<SM>, ug < 148 * 4 ? ug : 148 * 4, 512, 0, s, *L, (const float*)part, w, G,
                 wstride, NB, total, rr ? int64_t(grid) : nwarps, rr ? kWV : 1, maxseg, out, kmax, kres, kslots,
                 knwarps, total);
}

}  // namespace

// Any score / weight row stride: K writes scores with scalar stores, V picks
// vector or scalar weight loads per launch (wvec).
bool pkv_fast_supported(const pkv_layer_t* L, int G, int64_t stride) {
  (void)stride;
  return L->pack_size == kP && L->head_dim == kD && L->block == kRows && G >= 1 && G <= 8;
}

int pkv_fast_fused_k(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
                     cudaStream_t s) {
  launch_k<false>(L, nblocks, q, G, scores, sstride, nullptr, nullptr, 0, s);
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_k_scores(fast)");
}

int64_t pkv_fast_v_scratch(const pkv_layer_t* L, int nblocks, int G) {
  const int grid = v_grid<false>(L, nblocks, G);
  const int64_t nwarps = int64_t(grid) * kWV;
  return v_part_floats(L, G > 4 ? v_slots(L, nblocks, grid) : v_maxseg(L, nblocks, nwarps), G, nwarps) * 4;
}

int pkv_fast_fused_v(const pkv_layer_t* L, int nblocks, const float* w, int G, int64_t wstride, float* out,
                     float* part, cudaStream_t s) {
  launch_v<false>(L, nblocks, w, G, wstride, out, part, nullptr, nullptr, 0, 0, s);
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_v_output(fast)");
}

// attention_decode: scores (q pre-scaled by 1/sqrt(d)) with their softmax
// statistics, then the V pass on exp(s - M) and a normalising finalize.
// Scratch: kmax [U][kslots][G], kres [U][G], then the V partials.
int64_t pkv_fast_attention_scratch(const pkv_layer_t* L, int nblocks, int G) {
  const int64_t U = int64_t(L->batch) * L->heads;
  const int64_t knw = int64_t(k_grid<true>(L, nblocks, G)) * kWK;
  const int kslots = v_maxseg(L, nblocks, knw);
  const int vg = v_grid<true>(L, nblocks, G);
  const int64_t vnw = int64_t(vg) * kWV;
  const int64_t kf = (U * kslots * G + U * G + 3) / 4 * 4;
  return (kf + v_part_floats(L, G > 4 ? v_slots(L, nblocks, vg) : v_maxseg(L, nblocks, vnw), G, vnw)) * 4;
}

int pkv_fast_attention(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
                       float* out, float* scratch, cudaStream_t s) {
  const int64_t U = int64_t(L->batch) * L->heads;
  const int64_t knw = int64_t(k_grid<true>(L, nblocks, G)) * kWK;
  const int kslots = v_maxseg(L, nblocks, knw);
  float* kmax = scratch;
  float* kres = kmax + U * kslots * G;
  float* vpart = scratch + (U * kslots * G + U * G + 3) / 4 * 4;
  launch_k<true>(L, nblocks, q, G, scores, sstride, kmax, kres, kslots, s);
  launch_v<true>(L, nblocks, scores, G, sstride, out, vpart, kmax, kres, kslots, knw, s);
  return pkv_cuda_status(cudaGetLastError(), "pkv_attention_decode(fast)");
}
