// attn_fused.cu — single-pass decode attention over the compressed store
// (SPEC.md:520-528 attention_decode, §8 f1), default format, sm_100a.
//
// One launch per layer: softmax(q·deq(K)ᵀ)·deq(V) with no [B, Hq, L] score
// round trip through HBM (flash-decoding over compressed blocks, PAPER.md:375
// "single decompress+compute launch").
//
//  * Work split: the layer's (unit, item) sequence, unit = (sequence, kv-head),
//    items = the unit's blocks followed by buffer / 32 chunks of 32 residue
//    rows, is cut into one contiguous equal-length range per warp of the grid
//    (fast_common.cuh warp_range); the block count comes from the device
//    counts (attn_split), so a decode graph's headroom adds no empty items.
//  * Each warp streams the K and V block of every block item through its own
//    shared-memory ring (PAIRED feed: K then V of the same block), decodes K
//    into the transpose tile, takes the scores on the int8 tensor cores
//    (exactly as fused_k_fast_kernel), and keeps an online softmax per query
//    head: running maximum M (log2 domain), l = sum p, z = sum p·z_V and the
//    V accumulators acc = sum p·s·code, all relative to M.  Rows go to V as
//    p_t = exp(s_t - M); the V block is decoded and multiplied exactly as in
//    fused_v_fast_kernel (x = p·s in 2 unsigned byte digits per block and
//    head, exact int32 tile sums).
//  * Residue chunks: the uncompressed fp16 staging rows in f32 SIMT, folded
//    into the same running state.
//  * Merge: each (unit, warp) segment writes (acc, z, l, M) to a partial slot;
//    attn_merge_kernel folds a unit's slots in slot order, out = sum
//    e^(M_s - M*) (acc_s + z_s) / sum e^(M_s - M*) l_s, deterministic
//    (SPEC.md:487,490).  (Having the warp that completes a unit's last
//    segment merge it, with per-unit arrival counters, left a serial tail at
//    the end of the kernel and measured slower.)
//  * One copy of the unrolled unpack serves the K and the V phase of an item.
#include "fast_common.cuh"

#include <mutex>
#include <vector>

namespace {

constexpr int kWA = 4;                // warps per CTA
constexpr int kTileA = 4 * 128 * 16;  // K transpose tile (8 KB); after the K MMAs: sbuf, frag, vtmp (below)
constexpr int kResRows = 32;          // residue rows per range item
#ifndef PKV_RBA  // ring bytes per warp (a K block is ~3.9 KB, a V block ~3.4 KB at the paper's rel)
#define PKV_RBA 5888
#endif
#ifndef PKV_NSA
#define PKV_NSA 4
#endif
#ifndef PKV_APF  // L2 prefetch distance in feed items (K and V alternate)
#define PKV_APF 2
#endif
#ifndef PKV_ADIAG  // diagnostics build: per-warp cycle counters into `out` (results wrong)
#define PKV_ADIAG 0
#endif
#ifndef PKV_AMINB2  // the same for G <= 8 (NG = 2: 3 CTAs per SM measured 1408 -> 1271 us on config E)
#define PKV_AMINB2 3
#endif
#ifndef PKV_AABS  // absolute bit addressing of staged blocks (fast_common.cuh dbase / abase)
#define PKV_AABS 1
#endif
#ifndef PKV_AREGC  // pack width constants in registers (1) or from the shared table (0)
#define PKV_AREGC 0
#endif
#ifndef PKV_AMINB  // CTAs per SM the register allocation must allow
#define PKV_AMINB 3
#endif
constexpr int kRBA = PKV_RBA, kNSA = PKV_NSA;
using FeedA = Feed<kRBA, kNSA, PKV_APF, true>;
constexpr int kPartA = kD + 4;  // acc[128], z, l, M (log2 domain), pad
constexpr size_t kWarpSmemA = (kTileA + FeedA::bytes() + 127) / 128 * 128;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ldcg_f(const float* p) { return __ldcg(p); }

// Items per unit: the blocks, then ceil(buffer / 32) residue chunks.
__host__ __device__ __forceinline__ int res_items(int buffer) { return (buffer + kResRows - 1) / kResRows; }

// The work split over the layer's (unit, item) sequence, from the DEVICE block
// counts: a decode graph sizes `NB` with headroom for blocks appended later
// (GraphedDecodeLoop, up to 16 block-sets), and splitting the empty items too
// put two real items on warps that could have had one.  Items per unit NI =
// NBd + RI with NBd = the largest nblk[b], clamped to [NB - kNbSlack, NB] (the
// host sizes the partial slots for that range).  Warp-collective.
constexpr int kNbSlack = 64;
#ifndef PKV_ACHUNKS  // work split: chunks per warp of the grid
#define PKV_ACHUNKS 1
#endif
struct ASplit {
  int NB, NI;
  int64_t total, nchunks;
};
__device__ __forceinline__ ASplit attn_split(const pkv_layer_t& L, int NB, int RI, int64_t nwarps, int lane) {
  int m = 0;
  for (int b = lane; b < L.batch; b += 32) m = max(m, L.nblk[b]);
  m = int(__reduce_max_sync(PKV_FULL, unsigned(m)));
  ASplit sp;
  sp.NB = max(max(min(NB, m), NB - kNbSlack), 0);
  sp.NI = sp.NB + RI;
  sp.total = int64_t(L.batch) * L.heads * sp.NI;
  const int64_t want = nwarps * PKV_ACHUNKS;
  sp.nchunks = want < sp.total ? want : (sp.total > 0 ? sp.total : 1);
  return sp;
}

template <int NG, int MB>  // NG = 1: G <= 4 (one digit tile / n-tile), 2: G <= 8; MB: CTAs per SM
__global__ void __launch_bounds__(kWA * 32, MB)
    attn_fused_kernel(pkv_layer_t L, const float* __restrict__ q, int G, int NBh, int RI,
                      float* __restrict__ part, int maxseg, float* __restrict__ out) {
  constexpr int GP = 4 * NG;     // padded heads
  constexpr int LPH = 32 / GP;   // writer lanes per head
  constexpr int TPL = 64 / LPH;  // rows per writer lane (8 or 16)
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int U = L.batch * L.heads, Hq = L.heads * G;
  uint4* lut = (uint4*)smem;
  init_lut(lut, threadIdx.x);
  uint8_t* wsm = smem + 256 + warp * kWarpSmemA;
  // the tile region, once the K MMAs have read it:
  uint8_t* tile = wsm;
  float* sbuf = (float*)wsm;                   // [GP][64] the item's scores, then p (until the item ends)
  uint8_t* frag = wsm + 2048;                  // [GP][2][64] V B operand
  float* vtmp = (float*)(wsm + 3072);          // [GP][128] a scalar-path / residue V sum (channel per lane)
  uint32_t* xdesc = (uint32_t*)(wsm + 3072);   // [512] scalar-path descriptors (before vtmp is written)
  float* qsm = (float*)(wsm + 3072);           // [G][128] residue chunks: the q copy (K step)
  FeedA F;
  F.init(wsm + kTileA, lane);
  F.evf = true;  // the partials stay in L2 for the merge
  __syncthreads();
  // decode loop (PDL): the prologue above overlaps the previous kernel (the
  // layer's append-flush); the tables, arena and staging rows it writes are
  // read only after it completes
  pdl_wait();
  pdl_launch();
  const ASplit sp = attn_split(L, NBh, RI, int64_t(gridDim.x) * kWA, lane);
  const int NB = sp.NB, NI = sp.NI;
  const int64_t total = sp.total, nchunks = sp.nchunks;
  F.NI = NI;
  const uint32_t tile_s = smem_u32(tile);
  const uint8_t* lutb = (const uint8_t*)lut;
  const uint32_t R0 = 128u * (lane >> 3) + 64u * (lane & 1) + ((lane >> 1) & 3);
  const uint32_t X = 4u * (lane & 1);
  const uint32_t st_even = 16u * ((R0 & ~7u) | ((R0 & 7u) ^ X));
  const uint32_t st_odd = 16u * ((R0 & ~7u) | (((R0 & 7u) | 4u) ^ X));
  const int64_t nwarps = int64_t(gridDim.x) * kWA, wid = int64_t(blockIdx.x) * kWA + warp;
  // Work split: the item sequence is cut into `nchunks` equal contiguous
  // ranges (chunks), chunk c on warp c mod nwarps (nchunks = nwarps: one
  // contiguous range per warp).  Partial slots are per (unit, chunk).  (Taking
  // chunks from an atomic counter measured slower: every chunk start pays the
  // directory, query-fragment and first-block latencies.)
  int64_t cw = 0;  // current chunk
  Range rg;
  // writer role (softmax step and the V B operand): head wh, rows wt0 .. wt0 + TPL - 1
  const int wh = lane / LPH, wt0 = (lane % LPH) * TPL;

#if PKV_Q2
  QFrag2<NG> Q;
#else
  QFrag<NG> Q;
#endif
  float acc[NG][16];
  float Mw = -INFINITY, lacc = 0.f, zacc = 0.f;  // writer head wh: running max (log2), sum p, sum p z
#pragma unroll
  for (int nt = 0; nt < NG; ++nt)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[nt][i] = 0.f;

  // ---- partial of unit u (this warp's segment), then the merge by the last arriver
  auto flush = [&](int u) {
    const int64_t w0 = warp_of(int64_t(u) * NI, total, nchunks);
    const int64_t w1 = warp_of(int64_t(u + 1) * NI - 1, total, nchunks);
    float* pp = part + (int64_t(u) * maxseg + (cw - w0)) * G * kPartA;
#pragma unroll
    for (int nt = 0; nt < NG; ++nt) {
      const int g = 4 * nt + tq;
      if (g < G) {
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4)
          *(float4*)(pp + g * kPartA + 16 * gi + 4 * i4) =
              make_float4(acc[nt][4 * i4], acc[nt][4 * i4 + 1], acc[nt][4 * i4 + 2], acc[nt][4 * i4 + 3]);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[nt][i] = 0.f;
    }
    float z = zacc, l = lacc;
#pragma unroll
    for (int o = 1; o < LPH; o <<= 1) {
      z += __shfl_xor_sync(PKV_FULL, z, o);
      l += __shfl_xor_sync(PKV_FULL, l, o);
    }
    if (lane % LPH == 0 && wh < G) {
      pp[wh * kPartA + kD] = z;
      pp[wh * kPartA + kD + 1] = l;
      pp[wh * kPartA + kD + 2] = Mw;
    }
    Mw = -INFINITY;
    lacc = zacc = 0.f;
    // attn_merge_kernel merges the unit's slots
  };

  // ---- softmax step over sbuf (raw scores of this item's rows, -inf for rows
  // without a token): new running maximum, p = exp(s - M) back into sbuf, l
  // and the acc / z rescale.  Returns nothing; sbuf then holds p.
  auto softmax_step = [&]() {
    __syncwarp();
    float s[TPL];
#pragma unroll
    for (int e4 = 0; e4 < TPL / 4; ++e4) {
      const float4 v = *(const float4*)(sbuf + wh * 64 + wt0 + 4 * e4);
      s[4 * e4] = v.x; s[4 * e4 + 1] = v.y; s[4 * e4 + 2] = v.z; s[4 * e4 + 3] = v.w;
    }
    float bm = -INFINITY;
#pragma unroll
    for (int e = 0; e < TPL; ++e) {
      if (wh >= G) s[e] = 0.f;  // padded heads: finite, never output
      bm = fmaxf(bm, s[e]);
    }
#pragma unroll
    for (int o = 1; o < LPH; o <<= 1) bm = fmaxf(bm, __shfl_xor_sync(PKV_FULL, bm, o));
    const float Mn = fmaxf(Mw, bm * kLog2e);
    const float alpha = exp2f(Mw - Mn);  // Mw = -inf: 0
    Mw = Mn;
    float ps = 0.f;
#pragma unroll
    for (int e = 0; e < TPL; ++e) {
      s[e] = exp2f(fmaf(s[e], kLog2e, -Mn));
      ps += s[e];
    }
    lacc = fmaf(lacc, alpha, ps);
    zacc *= alpha;
#pragma unroll
    for (int e4 = 0; e4 < TPL / 4; ++e4)
      *(float4*)(sbuf + wh * 64 + wt0 + 4 * e4) = make_float4(s[4 * e4], s[4 * e4 + 1], s[4 * e4 + 2], s[4 * e4 + 3]);
    // acc lanes (gi, tq) hold head 4nt + tq: its writer lanes start at (4nt + tq) * LPH
    if (__any_sync(PKV_FULL, alpha != 1.f)) {
#pragma unroll
      for (int nt = 0; nt < NG; ++nt) {
        const float a = __shfl_sync(PKV_FULL, alpha, (4 * nt + tq) * LPH);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[nt][i] *= a;
      }
    }
    __syncwarp();
  };

  // ---- add vtmp [GP][128] (a block / chunk result in channel-per-lane layout) into acc
  auto add_vtmp = [&]() {
    __syncwarp();
#pragma unroll
    for (int nt = 0; nt < NG; ++nt) {
#pragma unroll
      for (int i4 = 0; i4 < 4; ++i4) {
        const float4 v = *(const float4*)(vtmp + (4 * nt + tq) * kD + 16 * gi + 4 * i4);
        acc[nt][4 * i4] += v.x;
        acc[nt][4 * i4 + 1] += v.y;
        acc[nt][4 * i4 + 2] += v.z;
        acc[nt][4 * i4 + 3] += v.w;
      }
    }
    __syncwarp();
  };

  int cur_u = -1, b = 0, h = 0;
#if PKV_ADIAG
  long long dg[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // wait K, wait V, K phase, V phase, all, items, end refill, unit change
  const long long dg0 = clock64();
  long long dgt = 0;
  int nitems = 0;
#endif
#pragma unroll 1
  for (cw = wid; cw < nchunks; cw += nwarps) {
  rg = warp_range(total, cw, nchunks);
  const int nk = int(rg.b1 - rg.b0);
#if PKV_ADIAG
  nitems += nk;
#endif
  // feed indices continue across chunks (the ring's mbarrier phases do)
  const int fb = F.issued;
  F.base = fb;
  F.k0 = fb - 32;
  Cursor cs;
  cs.init(rg.b0, NI, L.heads);
  cur_u = -1;
  F.refill(L, 0, NB, rg, fb + 2 * nk, fb - 1, F.head, lane);

#pragma unroll 1
  for (int k = 0; k < nk; ++k, cs.step(1, NI, L.heads)) {
    const int u = cs.u, j = cs.j;
    if (u != cur_u) {
#if PKV_ADIAG
      const long long tu = clock64();
#endif
      if (cur_u >= 0) flush(cur_u);
      cur_u = u;
      b = cs.b;
      h = cs.h;
      build_qfrag<NG>(q + (int64_t(b) * Hq + int64_t(h) * G) * kD, G, lane, Q);
#if PKV_ADIAG
      dg[7] += clock64() - tu;
#endif
    }
    const int src = 8 * tq + gi;  // V: the chunk this lane decodes (row-group tq, channels 16gi ..)
    if (j < NB) {
      // ============================ block item: K phase, softmax step, V phase.
      // ONE decode loop serves both phases (ph 0: K codes into the transpose
      // tile; ph 1: V codes straight into the IMMA A operand), one copy of the
      // unrolled unpack in the hot loop.  (ncu shows ~1 no-instruction stall
      // per issue against ~0.17 for the K or V kernel either way.)
#pragma unroll 1
      for (int ph = 0; ph < 2; ++ph) {
        const uint8_t* gb;
        bool have;
#if PKV_ADIAG
        dgt = clock64();
#endif
        const uint32_t sb = F.wait(fb + 2 * k + ph, &gb, &have);
#if PKV_ADIAG
        { const long long t1 = clock64(); dg[ph] += t1 - dgt; dgt = t1; }
#endif
        if (!have) break;  // past the sequence's block count: K and V both absent
        auto phase = [&](auto bp, bool may_fast_v) {
          Chunk ch;
          bool fast;
          uint32_t bf[NG][4];
          float inv[NG];
          if (ph == 0) {
            fast = parse_chunk(bp, lane, lane, ch);
          } else {
            // B operand: x_t = p_t * s_t as 2 unsigned byte digits scaled per
            // (block, head) (fused_v_fast_kernel), z term sum p_t z_t in f32
            parse_load(bp, lane, src, ch);
            uint2 pr[TPL / 2];
#pragma unroll
            for (int e2 = 0; e2 < TPL / 2; ++e2) pr[e2] = ld64(bp + kPar + 4 * (wt0 + 2 * e2));
            float wc[TPL];
#pragma unroll
            for (int e4 = 0; e4 < TPL / 4; ++e4) {
              const float4 v = *(const float4*)(sbuf + wh * 64 + wt0 + 4 * e4);
              wc[4 * e4] = v.x; wc[4 * e4 + 1] = v.y; wc[4 * e4 + 2] = v.z; wc[4 * e4 + 3] = v.w;
            }
            float xs[TPL];
            float mx = 0.f;
            bool neg = false;
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
            fast = parse_verdict(__reduce_or_sync(PKV_FULL, flags), ch) && may_fast_v;
            parse_scan(lane, ch);
#pragma unroll
            for (int o = 1; o < LPH; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(PKV_FULL, mx, o));
            const float f = mx > 1e-30f ? __fdividef(65535.f, mx) : 0.f;
            const float invf = mx * (1.f / 65535.f);
            if (fast) {
#pragma unroll
              for (int e8 = 0; e8 < TPL / 8; ++e8) {
                uint32_t v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = min(__float_as_uint(__fmaf_rn(xs[8 * e8 + e], f, 8388608.f)), 0x4B00FFFFu);
                const uint32_t t01 = __byte_perm(v[0], v[1], 0x5140), t45 = __byte_perm(v[4], v[5], 0x5140);
                const uint32_t t23 = __byte_perm(v[2], v[3], 0x5140), t67 = __byte_perm(v[6], v[7], 0x5140);
                const uint32_t lo0 = __byte_perm(t01, t45, 0x5410), hi0 = __byte_perm(t01, t45, 0x7632);
                const uint32_t lo1 = __byte_perm(t23, t67, 0x5410), hi1 = __byte_perm(t23, t67, 0x7632);
                *(uint2*)(frag + (wh * 2 + 0) * 64 + wt0 + 8 * e8) = make_uint2(lo0, lo1);
                *(uint2*)(frag + (wh * 2 + 1) * 64 + wt0 + 8 * e8) = make_uint2(hi0, hi1);
              }
              __syncwarp();
#pragma unroll
              for (int nt = 0; nt < NG; ++nt) {
                const uint4 v = *(const uint4*)(frag + ((4 * nt + (gi >> 1)) * 2 + (gi & 1)) * 64 + 16 * tq);
                bf[nt][0] = v.x; bf[nt][1] = v.y; bf[nt][2] = v.z; bf[nt][3] = v.w;
                inv[nt] = __shfl_sync(PKV_FULL, invf, (4 * nt + tq) * LPH);
              }
            }
          }
          if (fast) {
            // lane walks chunk cidx: its own (K: the transpose tile's order) or
            // chunk 8tq + gi (V: the A fragment's order); minima of that chunk are in ch.mn
            const int cidx = ph ? src : lane;
#if PKV_AABS
            uint32_t bit = __shfl_sync(PKV_FULL, ch.bit, cidx) + abase(bp);
            const auto db = dbase(bp);
#else
            uint32_t bit = __shfl_sync(PKV_FULL, ch.bit, cidx);
            const auto db = bp;
#endif
            const uint2 nb = ph ? ld64(bp + kNib + 8 * src) : ch.nb;
            auto decode = [&](auto wide) {
              uint32_t wa = w16_of(nb, 0), wb = w16_of(nb, 1);
              PackLd A = pack_load<PKV_AREGC>(db, lutb, bit, wa), B = pack_load<PKV_AREGC>(db, lutb, bit + wa, wb);
#pragma unroll
              for (int mt = 0; mt < 8; ++mt) {
                uint32_t P[2][4];
                const int i2 = 2 * mt;
                const uint32_t bitA = bit, bitB = bit + wa;
                const uint32_t nbit = bitB + wb;
                uint32_t nwa = 0, nwb = 0;
                PackLd nA, nB;
                if (i2 < 14) {
                  nwa = w16_of(nb, i2 + 2);
                  nwb = w16_of(nb, i2 + 3);
                  nA = pack_load<PKV_AREGC>(db, lutb, nbit, nwa);
                  nB = pack_load<PKV_AREGC>(db, lutb, nbit + nwa, nwb);
                }
                pack_decode<decltype(wide)::value>(db, A, bitA, wa, min_rep(ch.mn, i2), P[0]);
                pack_decode<decltype(wide)::value>(db, B, bitB, wb, min_rep(ch.mn, i2 + 1), P[1]);
                bit = nbit;
                wa = nwa;
                wb = nwb;
                if (i2 < 14) {
                  A = nA;
                  B = nB;
                }
                if (ph == 0) {
                  *(uint4*)(tile + st_even + 128u * mt) = make_uint4(P[0][0], P[0][1], P[0][2], P[0][3]);
                  *(uint4*)(tile + st_odd + 128u * mt) = make_uint4(P[1][0], P[1][1], P[1][2], P[1][3]);
                } else {
#pragma unroll
                  for (int nt = 0; nt < NG; ++nt) {
                    int d[4] = {0, 0, 0, 0};
                    const uint32_t a0[4] = {P[0][0], P[1][0], P[0][1], P[1][1]};
                    imma_uu(d, a0, bf[nt][0], bf[nt][1]);
                    const uint32_t a1[4] = {P[0][2], P[1][2], P[0][3], P[1][3]};
                    imma_uu(d, a1, bf[nt][2], bf[nt][3]);
                    acc[nt][2 * mt] = fmaf(float(d[0] + 256 * d[1]), inv[nt], acc[nt][2 * mt]);
                    acc[nt][2 * mt + 1] = fmaf(float(d[2] + 256 * d[3]), inv[nt], acc[nt][2 * mt + 1]);
                  }
                }
              }
            };
            if (ch.wide) decode(std::true_type{});
            else decode(std::false_type{});
            __syncwarp();  // tile stores (K) / frag reads (V) done
            if (ph == 0) {
              // scores of rows 16g + tok(gi) (+8), heads tq (+4), into sbuf (row-group 0 of the tile)
              float* s0 = sbuf + tq * 64 + tok(gi);
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                int accU[NG][4], accS[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  accS[e] = 0;
#pragma unroll
                  for (int nu = 0; nu < NG; ++nu) accU[nu][e] = 0;
                }
                const uint32_t prA = ld32(bp + kPar + 4 * (16 * g + tok(gi)));
                const uint32_t prB = ld32(bp + kPar + 4 * (16 * g + tok(gi) + 8));
                const uint32_t a0 = tile_s + 16u * (128u * g + lane);
                const uint32_t a1 = tile_s + 16u * (128u * g + (lane ^ 4u) + 64u);
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                  uint32_t a[4];
                  ldsm_t(a, (jj < 2 ? a0 : a1) + 512u * (jj & 1));
                  k_mma<NG>(accU, accS, a, Q, jj);
                }
                if (g == 0) __syncwarp();  // every lane has read row-group 0 (sbuf's bytes)
                const float sA = h2f(prA & 0xffff), zA = h2f(prA >> 16);
                const float sB = h2f(prB & 0xffff), zB = h2f(prB >> 16);
                {
                  const float vA = k_val<NG>(accU, accS, Q, 0, 0);
                  const float vB = k_val<NG>(accU, accS, Q, 0, 1);
                  s0[16 * g] = fmaf(sA, vA * Q.inv[0], zA * Q.qs[0]);
                  s0[16 * g + 8] = fmaf(sB, vB * Q.inv[0], zB * Q.qs[0]);
                }
                if (NG == 2) {
                  const float vA = k_val<NG>(accU, accS, Q, NG - 1, 0);
                  const float vB = k_val<NG>(accU, accS, Q, NG - 1, 1);
                  s0[256 + 16 * g] = fmaf(sA, vA * Q.inv[1], zA * Q.qs[1]);
                  s0[256 + 16 * g + 8] = fmaf(sB, vB * Q.inv[1], zB * Q.qs[1]);
                }
              }
            }
          } else if (ph == 0) {
            // scalar K (rare): lane computes rows lane and lane + 32 for every head
            const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * kD;
            const uint8_t* bg = gptr(bp);
            build_desc(ch, lane, xdesc);
#pragma unroll 1
            for (int half = 0; half < 2; ++half) {
              const int tt = lane + 32 * half, rgp = tt >> 4, t16 = tt & 15;
              const uint32_t prr = ld32(bg + kPar + 4 * tt);
              const float s = h2f(prr & 0xffff), z = h2f(prr >> 16);
#pragma unroll 1
              for (int g = 0; g < GP; ++g) {
                float a = 0.f, qsum = 0.f;
                if (g < G) {
#pragma unroll 1
                  for (int pos = 0; pos < 128; ++pos) {
                    const uint32_t d = xdesc[rgp * 128 + pos];
                    const uint32_t wd = d >> 18;
                    const float code = float(pack_min(bg, rgp * 128 + pos) + field_at(bg, (d & 0x3ffffu) + t16 * wd, wd));
                    const float qc = qu[g * kD + kpos_to_col(pos, kD)];
                    a = fmaf(code, qc, a);
                    qsum += qc;
                  }
                }
                sbuf[g * 64 + tt] = fmaf(s, a, z * qsum);
              }
            }
          } else {
            // scalar V (rare): lane owns channels lane + 32 q4, all 64 rows, every
            // head; the block's sum goes through vtmp into acc
            const uint8_t* bg = gptr(bp);
            build_desc(ch, lane, xdesc);
            float sacc[GP][4];
#pragma unroll
            for (int g = 0; g < GP; ++g)
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) sacc[g][q4] = 0.f;
#pragma unroll 1
            for (int r = 0; r < kRows; ++r) {
              const uint32_t prr = ld32(bg + kPar + 4 * r);
              const float s = h2f(prr & 0xffff);
              float ws[GP];
#pragma unroll
              for (int g = 0; g < GP; ++g) ws[g] = sbuf[g * 64 + r] * s;
              const int rgp = r >> 4, tt = r & 15;
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) {
                const int c = lane + 32 * q4;
                const uint32_t dd = xdesc[rgp * 128 + c];
                const uint32_t wd = dd >> 18;
                const float code = float(pack_min(bg, rgp * 128 + c) + field_at(bg, (dd & 0x3ffffu) + tt * wd, wd));
#pragma unroll
                for (int g = 0; g < GP; ++g) sacc[g][q4] = fmaf(ws[g], code, sacc[g][q4]);
              }
            }
            __syncwarp();
#pragma unroll
            for (int g = 0; g < GP; ++g)
#pragma unroll
              for (int q4 = 0; q4 < 4; ++q4) vtmp[g * kD + lane + 32 * q4] = sacc[g][q4];
            add_vtmp();
          }
        };
        if (gb)
          phase(gb, false);  // too large for the ring: read in place (V takes the scalar path)
        else
          phase(sb, true);
        if (ph == 0) {
          // the K block's ring bytes are free: top up the feed while V runs
          F.refill(L, 0, NB, rg, fb + 2 * nk, fb + 2 * k, F.tail_after(fb + 2 * k), lane);
          softmax_step();
        }
#if PKV_ADIAG
        dg[2 + ph] += clock64() - dgt;
#endif
      }
    } else {
      // ============================ residue chunk: staged rows r0 .. r0 + 31 (fp16, f32 SIMT)
      const int r0 = (j - NB) * kResRows;
      const int nres = min(L.nres[b] - r0, kResRows);
      if (nres > 0) {
        const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * kD;
        __syncwarp();
        for (int i = lane; i < G * kD / 4; i += 32) reinterpret_cast<float4*>(qsm)[i] = reinterpret_cast<const float4*>(qu)[i];
        __syncwarp();
        float a[GP];
#pragma unroll
        for (int g = 0; g < GP; ++g) a[g] = 0.f;
        if (lane < nres) {
          const uint4* kr = reinterpret_cast<const uint4*>(L.stage + (int64_t(u) * L.buffer + r0 + lane) * kD);
#pragma unroll 2
          for (int c8 = 0; c8 < kD / 8; ++c8) {
            const uint4 v = kr[c8];
            const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float x0 = h2f(wv[e] & 0xffff), x1 = h2f(wv[e] >> 16);
#pragma unroll
              for (int g = 0; g < GP; ++g)
                if (g < G) {
                  const float2 qv = *reinterpret_cast<const float2*>(qsm + g * kD + 8 * c8 + 2 * e);
                  a[g] = fmaf(x1, qv.y, fmaf(x0, qv.x, a[g]));
                }
            }
          }
        }
        __syncwarp();  // qsm reads done (sbuf and vtmp follow)
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          sbuf[g * 64 + lane] = lane < nres ? a[g] : -INFINITY;
          sbuf[g * 64 + 32 + lane] = -INFINITY;
        }
        softmax_step();
        // out[g][c] += sum_t p[g][t] v[t][c], lane owns channels 4 lane .. + 3
        float av[GP][4];
#pragma unroll
        for (int g = 0; g < GP; ++g) av[g][0] = av[g][1] = av[g][2] = av[g][3] = 0.f;
        const uint16_t* vr = L.stage + ((int64_t(U) + u) * L.buffer + r0) * kD + 4 * lane;
#pragma unroll 2
        for (int t = 0; t < nres; ++t) {
          const uint2 v = *reinterpret_cast<const uint2*>(vr + int64_t(t) * kD);
          const float x0 = h2f(v.x & 0xffff), x1 = h2f(v.x >> 16), x2 = h2f(v.y & 0xffff), x3 = h2f(v.y >> 16);
#pragma unroll
          for (int g = 0; g < GP; ++g) {
            const float p = sbuf[g * 64 + t];
            av[g][0] = fmaf(p, x0, av[g][0]);
            av[g][1] = fmaf(p, x1, av[g][1]);
            av[g][2] = fmaf(p, x2, av[g][2]);
            av[g][3] = fmaf(p, x3, av[g][3]);
          }
        }
        __syncwarp();
#pragma unroll
        for (int g = 0; g < GP; ++g) *(float4*)(vtmp + g * kD + 4 * lane) = make_float4(av[g][0], av[g][1], av[g][2], av[g][3]);
        add_vtmp();
      }
    }
#if PKV_ADIAG
    const long long tr = clock64();
#endif
    F.refill(L, 0, NB, rg, fb + 2 * nk, fb + 2 * k + 1, F.tail_after(fb + 2 * k + 1), lane);
#if PKV_ADIAG
    dg[6] += clock64() - tr;
#endif
  }
  if (cur_u >= 0) flush(cur_u);
  }
#if PKV_ADIAG
  __syncwarp();
  if (lane == 0) {
    long long* dbg = reinterpret_cast<long long*>(out) + 8 * wid;
    dg[4] = clock64() - dg0;
    dg[5] = nitems;
    for (int i = 0; i < 8; ++i) dbg[i] = dg[i];
  }
#endif
}

// The unit's slot partials merged in slot order (deterministic): one CTA of
// 128 x kMQ threads per (unit, head); thread (q, c) folds slots q, q + kMQ, ...
// of channel c with an online maximum, then the kMQ groups are combined in a
// fixed order.  out = sum_s e^(M_s - M*) (acc_s + z_s) / sum_s e^(M_s - M*) l_s.
constexpr int kMQ = 8;
__global__ void __launch_bounds__(128 * kMQ) attn_merge_kernel(pkv_layer_t L, int G, int NBh, int RI,
                                                             int64_t fwarps, const float* __restrict__ part,
                                                             int maxseg, float* __restrict__ out) {
  __shared__ float rm[kMQ], rz[kMQ], rl[kMQ], ro[kMQ][kD];
  const int c = threadIdx.x & 127, qq = threadIdx.x >> 7;
  const int U = L.batch * L.heads, Hq = L.heads * G;
  pdl_wait();  // the partials of attn_fused_kernel
  pdl_launch();
  // the attention kernel's split (fwarps: its warps), from the same device counts
  const ASplit sp = attn_split(L, NBh, RI, fwarps, threadIdx.x & 31);
  const int NI = sp.NI;
  const int64_t total = sp.total, nwarps = sp.nchunks;
  for (int ug = blockIdx.x; ug < U * G; ug += gridDim.x) {
    const int u = ug / G, g = ug - u * G;
    const int64_t w0 = warp_of(int64_t(u) * NI, total, nwarps), w1 = warp_of(int64_t(u + 1) * NI - 1, total, nwarps);
    const int ns = int(w1 - w0 + 1);
    const float* pg = part + (int64_t(u) * maxseg * G + g) * kPartA;
    const int64_t st = int64_t(G) * kPartA;
    float m = -INFINITY, o = 0.f, z = 0.f, l = 0.f;
    auto fold = [&](float Ms, float a, float zs, float ls) {
      if (Ms > m) {
        const float sc = exp2f(m - Ms);  // m = -inf: 0
        o *= sc;
        z *= sc;
        l *= sc;
        m = Ms;
      }
      const float e = Ms == -INFINITY ? 0.f : exp2f(Ms - m);
      o = fmaf(e, a, o);
      z = fmaf(e, zs, z);
      l = fmaf(e, ls, l);
    };
    // eight slots' loads in flight per round (one round for <= 64 slots): a partial
    // round loads a valid slot again (index clamped, loads unconditional) and folds
    // it as empty (M = -inf is a no-op), instead of a tail of dependent single-slot loads
    for (int s = qq; s < ns; s += 8 * kMQ) {
      float Mv[8], av[8], zv[8], lv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float* ps = pg + min(s + i * kMQ, ns - 1) * st;
        Mv[i] = ps[kD + 2];
        av[i] = ps[c];
        zv[i] = ps[kD];
        lv[i] = ps[kD + 1];
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) fold(s + i * kMQ < ns ? Mv[i] : -INFINITY, av[i], zv[i], lv[i]);
    }
    ro[qq][c] = o;
    if (c == 0) {
      rm[qq] = m;
      rz[qq] = z;
      rl[qq] = l;
    }
    __syncthreads();
    if (qq == 0) {
      float M = -INFINITY;
#pragma unroll
      for (int i = 0; i < kMQ; ++i) M = fmaxf(M, rm[i]);
      float O = 0.f, Z = 0.f, Lw = 0.f;
#pragma unroll
      for (int i = 0; i < kMQ; ++i) {
        const float e = rm[i] == -INFINITY ? 0.f : exp2f(rm[i] - M);
        O = fmaf(e, ro[i][c], O);
        Z = fmaf(e, rz[i], Z);
        Lw = fmaf(e, rl[i], Lw);
      }
      const int b = u / L.heads, h = u - b * L.heads;
      out[(int64_t(b) * Hq + int64_t(h) * G + g) * kD + c] = Lw > 0.f ? (O + Z) / Lw : 0.f;
    }
    __syncthreads();
  }
}

constexpr size_t a_smem_bytes() { return 256 + kWA * kWarpSmemA; }

// resident CTAs per device for each instantiation (queried once per device)
template <class K>
int attn_grid_cap(K kernel) {
  struct Cap {
    const void* k;
    int dev, cap;
  };
  static std::mutex mu;
  static std::vector<Cap> caps;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lock(mu);
    for (const Cap& c : caps)
      if (c.k == (const void*)kernel && c.dev == dev) return c.cap;
  }
  int nsm = 0, per = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(a_smem_bytes()));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kWA * 32, a_smem_bytes());
  const int cap = max(1, per) * nsm;
  std::lock_guard<std::mutex> lock(mu);
  caps.push_back({(const void*)kernel, dev, cap});
  return cap;
}

struct AttnPlan {
  int NB, NI, grid, maxseg, G, mb;
  int64_t total, nchunks;
};

AttnPlan attn_plan(const pkv_layer_t* L, int nblocks, int G) {
  AttnPlan p;
  p.G = G;
  p.NB = max(0, nblocks);
  p.NI = p.NB + res_items(L->buffer);
  const int64_t U = int64_t(L->batch) * L->heads;
  p.total = U * p.NI;
  // G <= 4: 3 CTAs per SM (168 registers, no spills) while the items fit one
  // per warp, else 4 (128 registers, a few spills) so a layer with more items
  // than 12 warps per SM hold runs fewer rounds (config C 716 -> 744 tokens/s)
  int cap = G <= 4 ? attn_grid_cap(attn_fused_kernel<1, PKV_AMINB>) : attn_grid_cap(attn_fused_kernel<2, PKV_AMINB2>);
  p.mb = G <= 4 ? PKV_AMINB : PKV_AMINB2;
  if (G <= 4 && p.total > int64_t(cap) * kWA) {
    cap = attn_grid_cap(attn_fused_kernel<1, 4>);
    p.mb = 4;
  }
  const int64_t want = (p.total + kWA - 1) / kWA;
  p.grid = int(want < 1 ? 1 : (want < cap ? want : cap));
  const int64_t nwarps = int64_t(p.grid) * kWA;
  p.nchunks = nwarps * PKV_ACHUNKS < p.total ? nwarps * PKV_ACHUNKS : (p.total > 0 ? p.total : 1);
  // slots per unit: the most chunks whose ranges can meet one unit, over every
  // device block count the kernels may split by (attn_split)
  const int RI = res_items(L->buffer);
  p.maxseg = 1;
  for (int nb = max(0, p.NB - kNbSlack); nb <= p.NB; ++nb) {
    const int64_t ni = nb + RI, tot = U * ni;
    const int64_t nch = nwarps * PKV_ACHUNKS < tot ? nwarps * PKV_ACHUNKS : (tot > 0 ? tot : 1);
    const int64_t len_min = tot / nch;
    const int ms = len_min == 0 ? int(ni < nch ? ni : nch) + 1 : int((ni + len_min - 1) / len_min + 1);
    p.maxseg = max(p.maxseg, ms);
  }
  return p;
}

}  // namespace

// Scratch: 16 reserved bytes, then the partials [U][maxseg][G][kPartA] f32.
int64_t pkv_fast_attention1_scratch(const pkv_layer_t* L, int nblocks, int G) {
  const AttnPlan p = attn_plan(L, nblocks, G);
  const int64_t U = int64_t(L->batch) * L->heads;
  return 16 + U * p.maxseg * G * kPartA * 4;
}

int pkv_fast_attention1(const pkv_layer_t* L, int nblocks, const float* q, int G, float* out, void* scratch,
                        cudaStream_t s) {
  const AttnPlan p = attn_plan(L, nblocks, G);
  const int64_t U = int64_t(L->batch) * L->heads;
  float* part = (float*)((uint8_t*)scratch + 16);
  const int RI = res_items(L->buffer);
  cudaError_t e;
  if (G > 4)
    e = pkv_launch_pdl(attn_fused_kernel<2, PKV_AMINB2>, p.grid, kWA * 32, a_smem_bytes(), s, *L, q, G, p.NB, RI, part,
                       p.maxseg, out);
  else if (p.mb == 4)
    e = pkv_launch_pdl(attn_fused_kernel<1, 4>, p.grid, kWA * 32, a_smem_bytes(), s, *L, q, G, p.NB, RI, part,
                       p.maxseg, out);
  else
    e = pkv_launch_pdl(attn_fused_kernel<1, PKV_AMINB>, p.grid, kWA * 32, a_smem_bytes(), s, *L, q, G, p.NB, RI,
                       part, p.maxseg, out);
  if (e != cudaSuccess) return pkv_cuda_status(e, "pkv_attention_decode(single pass)");
  if (!PKV_ADIAG) {
    const int ug = int(U) * G;
    e = pkv_launch_pdl(attn_merge_kernel, ug < 148 * 2 ? ug : 148 * 2, 128 * kMQ, 0, s, *L, G, p.NB, RI,
                       int64_t(p.grid) * kWA, (const float*)part, p.maxseg, out);
    if (e != cudaSuccess) return pkv_cuda_status(e, "pkv_attention_decode(single pass): merge");
  }
  return pkv_cuda_status(cudaGetLastError(), "pkv_attention_decode(single pass)");
}
