// attn_fused.cu — single-pass decode attention over the compressed store
// (SPEC.md:520-528 attention_decode, §8 f1), default format, sm_100a.
//
// One launch per layer: softmax(q·deq(K)ᵀ)·deq(V) with no [B, Hq, L] score
// round trip through HBM (flash-decoding over compressed blocks, PAPER.md:375
// "single decompress+compute launch").
//
//  * Work split: the layer's (unit, item) sequence, unit = (sequence, kv-head),
//    items = the unit's NB blocks followed by kResItems chunks of 32 residue
//    rows, is cut into one contiguous equal-length range per warp of the grid
//    (fast_common.cuh warp_range).
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
//    the warp that completes a unit's last segment (per-unit arrival counter)
//    merges the unit's slots in slot order, out = sum e^(M_s - M*) (acc_s +
//    z_s) / sum e^(M_s - M*) l_s, and resets the counter.  The result does not
//    depend on arrival order (deterministic).
#include "fast_common.cuh"

#include <mutex>
#include <vector>

namespace {

constexpr int kWA = 4;                // warps per CTA
constexpr int kTileA = 4 * 128 * 16;  // K transpose tile (8 KB); V phase: vtmp [8][128] f32 + frag [8][2][64]
constexpr int kResRows = 32;          // residue rows per range item
#ifndef PKV_RBA  // ring bytes per warp: one K+V block pair (~7.3 KB at the paper's rel) plus the next K
#define PKV_RBA 8192
#endif
#ifndef PKV_NSA
#define PKV_NSA 4
#endif
#ifndef PKV_APF  // L2 prefetch distance in feed items (K and V alternate)
#define PKV_APF 2
#endif
#ifndef PKV_AMINB  // CTAs per SM the register allocation must allow (shared memory allows 3)
#define PKV_AMINB 3
#endif
constexpr int kRBA = PKV_RBA, kNSA = PKV_NSA;
using FeedA = Feed<kRBA, kNSA, PKV_APF, true>;
constexpr int kPartA = kD + 4;  // acc[128], z, l, M (log2 domain), pad
constexpr size_t kWarpSmemA = (kTileA + 2048 + FeedA::bytes() + 127) / 128 * 128;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ldcg_f(const float* p) { return __ldcg(p); }

// Items per unit: the blocks, then ceil(buffer / 32) residue chunks.
__host__ __device__ __forceinline__ int res_items(int buffer) { return (buffer + kResRows - 1) / kResRows; }

template <int NG>  // NG = 1: G <= 4 (one digit tile / n-tile), 2: G <= 8
__global__ void __launch_bounds__(kWA * 32, PKV_AMINB)
    attn_fused_kernel(pkv_layer_t L, const float* __restrict__ q, int G, int NB, int NI, int64_t total,
                      float* __restrict__ part, int maxseg, int* __restrict__ cnt, float* __restrict__ out) {
  constexpr int GP = 4 * NG;     // padded heads
  constexpr int LPH = 32 / GP;   // writer lanes per head
  constexpr int TPL = 64 / LPH;  // rows per writer lane (8 or 16)
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gi = lane >> 2, tq = lane & 3;
  const int U = L.batch * L.heads, Hq = L.heads * G;
  uint4* lut = (uint4*)smem;
  init_lut(lut, threadIdx.x);
  uint8_t* wsm = smem + 256 + warp * kWarpSmemA;
  uint8_t* tile = wsm;
  float* vtmp = (float*)wsm;                   // [GP][128] (V phase)
  uint8_t* frag = wsm + 4096;                  // [GP][2][64] (V phase)
  uint32_t* vdesc = (uint32_t*)(wsm + 5120);   // [512] scalar V path (V phase)
  float* qsm = (float*)(wsm + 4096);           // [G][128] residue chunks (q copy)
  float* sbuf = (float*)(wsm + kTileA);        // [GP][64] scores, then p
  FeedA F;
  F.init(wsm + kTileA + 2048, lane);
  F.NI = NI;
  __syncthreads();
  const uint32_t tile_s = smem_u32(tile);
  const uint8_t* lutb = (const uint8_t*)lut;
  const uint32_t R0 = 128u * (lane >> 3) + 64u * (lane & 1) + ((lane >> 1) & 3);
  const uint32_t X = 4u * (lane & 1);
  const uint32_t st_even = 16u * ((R0 & ~7u) | ((R0 & 7u) ^ X));
  const uint32_t st_odd = 16u * ((R0 & ~7u) | (((R0 & 7u) | 4u) ^ X));
  const int64_t nwarps = int64_t(gridDim.x) * kWA, wid = int64_t(blockIdx.x) * kWA + warp;
  const Range rg = warp_range(total, wid, nwarps);
  const int nk = int(rg.b1 - rg.b0);
  // writer role (softmax step and the V B operand): head wh, rows wt0 .. wt0 + TPL - 1
  const int wh = lane / LPH, wt0 = (lane % LPH) * TPL;

  QFrag<NG> Q;
  float acc[NG][16];
  float Mw = -INFINITY, lacc = 0.f, zacc = 0.f;  // writer head wh: running max (log2), sum p, sum p z
#pragma unroll
  for (int nt = 0; nt < NG; ++nt)
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[nt][i] = 0.f;

  // ---- partial of unit u (this warp's segment), then the merge by the last arriver
  auto flush = [&](int u) {
    const int64_t w0 = warp_of(int64_t(u) * NI, total, nwarps);
    const int64_t w1 = warp_of(int64_t(u + 1) * NI - 1, total, nwarps);
    float* pp = part + (int64_t(u) * maxseg + (wid - w0)) * G * kPartA;
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
    __threadfence();
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atomicAdd(&cnt[u], 1) == int(w1 - w0);
    last = __shfl_sync(PKV_FULL, last, 0);
    if (!last) return;
    __threadfence();
    const int ns = int(w1 - w0 + 1);
    const float* pu = part + int64_t(u) * maxseg * G * kPartA;
    const int64_t st = int64_t(G) * kPartA;
    const int b = u / L.heads, h = u - b * L.heads;
    for (int g = 0; g < G; ++g) {
      float m = -INFINITY;
      for (int s = lane; s < ns; s += 32) m = fmaxf(m, ldcg_f(pu + s * st + g * kPartA + kD + 2));
      m = warp_max(m);
      float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
      float zs = 0.f, ls = 0.f;
#pragma unroll 4
      for (int s = 0; s < ns; ++s) {
        const float* ps = pu + s * st + g * kPartA;
        const float Ms = ldcg_f(ps + kD + 2);
        const float e = Ms == -INFINITY ? 0.f : exp2f(Ms - m);
        const float4 a = __ldcg((const float4*)(ps + 4 * lane));
        o.x = fmaf(e, a.x, o.x);
        o.y = fmaf(e, a.y, o.y);
        o.z = fmaf(e, a.z, o.z);
        o.w = fmaf(e, a.w, o.w);
        zs = fmaf(e, ldcg_f(ps + kD), zs);
        ls = fmaf(e, ldcg_f(ps + kD + 1), ls);
      }
      const float inv = ls > 0.f ? 1.f / ls : 0.f;
      *(float4*)(out + (int64_t(b) * Hq + int64_t(h) * G + g) * kD + 4 * lane) =
          make_float4((o.x + zs) * inv, (o.y + zs) * inv, (o.z + zs) * inv, (o.w + zs) * inv);
    }
    if (lane == 0) cnt[u] = 0;  // ready for the next launch
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

  Cursor cs;
  cs.init(rg.b0, NI, L.heads);
  int cur_u = -1, b = 0, h = 0;
  F.refill(L, 0, NB, rg, 2 * nk, -1, 0u, lane);

#pragma unroll 1
  for (int k = 0; k < nk; ++k, cs.step(1, NI, L.heads)) {
    const int u = cs.u, j = cs.j;
    if (u != cur_u) {
      if (cur_u >= 0) flush(cur_u);
      cur_u = u;
      b = cs.b;
      h = cs.h;
      build_qfrag<NG>(q + (int64_t(b) * Hq + int64_t(h) * G) * kD, G, lane, Q);
    }
    // ================================================================ K phase
    const uint8_t* gk;
    bool have_k;
    const uint32_t kblk = F.wait(2 * k, &gk, &have_k);
    bool rows = false;  // the item holds at least one token
    int nres = 0, r0 = 0;
    if (j < NB) {
      if (have_k) {
        rows = true;
        Chunk ch;
        auto fast_block = [&](auto bp) {
          auto decode_packs = [&](auto wide) {
            uint32_t bit = ch.bit;
            uint32_t wa = w16_of(ch.nb, 0), wb = w16_of(ch.nb, 1);
            PackLd A = pack_load<PKV_KREGC>(bp, lutb, bit, wa), B = pack_load<PKV_KREGC>(bp, lutb, bit + wa, wb);
#pragma unroll
            for (int i2 = 0; i2 < 16; i2 += 2) {
              const uint32_t bitA = bit, bitB = bit + wa;
              const uint32_t nbit = bitB + wb;
              uint32_t nwa = 0, nwb = 0;
              PackLd nA, nB;
              if (i2 < 14) {
                nwa = w16_of(ch.nb, i2 + 2);
                nwb = w16_of(ch.nb, i2 + 3);
                nA = pack_load<PKV_KREGC>(bp, lutb, nbit, nwa);
                nB = pack_load<PKV_KREGC>(bp, lutb, nbit + nwa, nwb);
              }
              uint32_t ra[4], rb[4];
              pack_decode<decltype(wide)::value>(bp, A, bitA, wa, min_rep(ch.mn, i2), ra);
              pack_decode<decltype(wide)::value>(bp, B, bitB, wb, min_rep(ch.mn, i2 + 1), rb);
              *(uint4*)(tile + st_even + 128u * (i2 >> 1)) = make_uint4(ra[0], ra[1], ra[2], ra[3]);
              *(uint4*)(tile + st_odd + 128u * (i2 >> 1)) = make_uint4(rb[0], rb[1], rb[2], rb[3]);
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
          uint32_t prm[4][2];
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            prm[g][0] = ld32(bp + kPar + 4 * (16 * g + tok(gi)));
            prm[g][1] = ld32(bp + kPar + 4 * (16 * g + tok(gi) + 8));
          }
          __syncwarp();
          float* s0 = sbuf + tq * 64 + tok(gi);  // rows 16g + tok(gi) (+8) of head tq (+4)
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            int accU[NG][4], accS[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              accS[e] = 0;
#pragma unroll
              for (int nu = 0; nu < NG; ++nu) accU[nu][e] = 0;
            }
            const uint32_t a0 = tile_s + 16u * (128u * g + lane);
            const uint32_t a1 = tile_s + 16u * (128u * g + (lane ^ 4u) + 64u);
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              uint32_t a[4];
              ldsm_t(a, (jj < 2 ? a0 : a1) + 512u * (jj & 1));
#pragma unroll
              for (int nu = 0; nu < NG; ++nu) imma_uu(accU[nu], a, Q.u[nu][jj][0], Q.u[nu][jj][1]);
              imma_us(accS, a, Q.s[jj][0], Q.s[jj][1]);
            }
            const float sA = h2f(prm[g][0] & 0xffff), zA = h2f(prm[g][0] >> 16);
            const float sB = h2f(prm[g][1] & 0xffff), zB = h2f(prm[g][1] >> 16);
            {
              const float vA = fmaf(65536.f, float(accS[0]), float(accU[0][0] + 256 * accU[0][1]));
              const float vB = fmaf(65536.f, float(accS[2]), float(accU[0][2] + 256 * accU[0][3]));
              s0[16 * g] = fmaf(sA, vA * Q.inv[0], zA * Q.qs[0]);
              s0[16 * g + 8] = fmaf(sB, vB * Q.inv[0], zB * Q.qs[0]);
            }
            if (NG == 2) {
              const float vA = fmaf(65536.f, float(accS[1]), float(accU[NG - 1][0] + 256 * accU[NG - 1][1]));
              const float vB = fmaf(65536.f, float(accS[3]), float(accU[NG - 1][2] + 256 * accU[NG - 1][3]));
              s0[256 + 16 * g] = fmaf(sA, vA * Q.inv[1], zA * Q.qs[1]);
              s0[256 + 16 * g + 8] = fmaf(sB, vB * Q.inv[1], zB * Q.qs[1]);
            }
          }
          __syncwarp();  // tile reads done
        };
        bool fast;
        if (gk == nullptr) {
          fast = parse_chunk(kblk, lane, lane, ch);
          if (fast) fast_block(kblk);
        } else {
          fast = parse_chunk(gk, lane, lane, ch);
          if (fast) fast_block(gk);
        }
        if (!fast) {
          // scalar path (rare): lane computes rows lane and lane + 32 for every head
          const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * kD;
          uint32_t* desc = (uint32_t*)tile;
          const uint8_t* bg = gk ? gk : gptr(kblk);
          if (gk) parse_chunk(bg, lane, lane, ch);
          build_desc(ch, lane, desc);
#pragma unroll 1
          for (int half = 0; half < 2; ++half) {
            const int tt = lane + 32 * half, rgp = tt >> 4, t16 = tt & 15;
            const uint32_t pr = ld32(bg + kPar + 4 * tt);
            const float s = h2f(pr & 0xffff), z = h2f(pr >> 16);
#pragma unroll 1
            for (int g = 0; g < GP; ++g) {
              float a = 0.f, qsum = 0.f;
              if (g < G) {
#pragma unroll 1
                for (int pos = 0; pos < 128; ++pos) {
                  const uint32_t d = desc[rgp * 128 + pos];
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
          __syncwarp();
        }
      }
    } else {
      // residue chunk: staged rows r0 .. r0 + 31 of the unit (fp16, f32 SIMT)
      r0 = (j - NB) * kResRows;
      nres = min(L.nres[b] - r0, kResRows);
      if (nres > 0) {
        rows = true;
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
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          sbuf[g * 64 + lane] = lane < nres ? a[g] : -INFINITY;
          sbuf[g * 64 + 32 + lane] = -INFINITY;
        }
      }
    }
    // the K block's ring bytes are free: top up the feed while V runs
    F.refill(L, 0, NB, rg, 2 * nk, 2 * k, F.tail_after(2 * k), lane);
    if (rows) softmax_step();

    // ================================================================ V phase
    const uint8_t* gv;
    bool have_v;
    const uint32_t vsb = F.wait(2 * k + 1, &gv, &have_v);
    if (rows && j < NB && have_v) {
      auto process = [&](auto blk, bool may_fast) {
        Chunk ch;
        const int src = 8 * tq + gi;
        parse_load(blk, lane, src, ch);
        uint2 pr[TPL / 2];
#pragma unroll
        for (int e2 = 0; e2 < TPL / 2; ++e2) pr[e2] = ld64(blk + kPar + 4 * (wt0 + 2 * e2));
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
        const bool fast = parse_verdict(__reduce_or_sync(PKV_FULL, flags), ch) && may_fast;
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
          uint32_t bf[NG][4];
          float inv[NG];
#pragma unroll
          for (int nt = 0; nt < NG; ++nt) {
            const uint4 v = *(const uint4*)(frag + ((4 * nt + (gi >> 1)) * 2 + (gi & 1)) * 64 + 16 * tq);
            bf[nt][0] = v.x; bf[nt][1] = v.y; bf[nt][2] = v.z; bf[nt][3] = v.w;
            inv[nt] = __shfl_sync(PKV_FULL, invf, (4 * nt + tq) * LPH);
          }
          uint32_t bit = __shfl_sync(PKV_FULL, ch.bit, src);
          const uint2 nb = ld64(blk + kNib + 8 * src);
          const uint32_t (&mn)[8] = ch.mn;
          auto decode_mma = [&](auto wide) {
            uint32_t wa = w16_of(nb, 0), wb = w16_of(nb, 1);
            PackLd A = pack_load(blk, lutb, bit, wa), B = pack_load(blk, lutb, bit + wa, wb);
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
              uint32_t P[2][4];
              {
                const int i2 = 2 * mt;
                const uint32_t bitA = bit, bitB = bit + wa;
                const uint32_t nbit = bitB + wb;
                uint32_t nwa = 0, nwb = 0;
                PackLd nA, nB;
                if (i2 < 14) {
                  nwa = w16_of(nb, i2 + 2);
                  nwb = w16_of(nb, i2 + 3);
                  nA = pack_load(blk, lutb, nbit, nwa);
                  nB = pack_load(blk, lutb, nbit + nwa, nwb);
                }
                pack_decode<decltype(wide)::value>(blk, A, bitA, wa, min_rep(mn, i2), P[0]);
                pack_decode<decltype(wide)::value>(blk, B, bitB, wb, min_rep(mn, i2 + 1), P[1]);
                bit = nbit;
                wa = nwa;
                wb = nwb;
                if (i2 < 14) {
                  A = nA;
                  B = nB;
                }
              }
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
          };
          if (ch.wide) decode_mma(std::true_type{});
          else decode_mma(std::false_type{});
          __syncwarp();  // frag reads done before the next block's tile stores
        } else {
          // scalar path (rare): lane owns channels lane + 32 q4, all 64 rows, every
          // head; the block's sum goes through vtmp into acc
          const uint8_t* bg = gptr(blk);
          build_desc(ch, lane, vdesc);
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
              const uint32_t dd = vdesc[rgp * 128 + c];
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
      if (gv)
        process(gv, false);
      else
        process(F.ring + (vsb - smem_u32(F.ring)), true);
    } else if (rows && j >= NB) {
      // residue chunk: out[g][c] += sum_t p[g][t] v[t][c], lane owns channels 4 lane .. + 3
      float a[GP][4];
#pragma unroll
      for (int g = 0; g < GP; ++g) a[g][0] = a[g][1] = a[g][2] = a[g][3] = 0.f;
      const uint16_t* vr = L.stage + ((int64_t(U) + u) * L.buffer + r0) * kD + 4 * lane;
#pragma unroll 2
      for (int t = 0; t < nres; ++t) {
        const uint2 v = *reinterpret_cast<const uint2*>(vr + int64_t(t) * kD);
        const float x0 = h2f(v.x & 0xffff), x1 = h2f(v.x >> 16), x2 = h2f(v.y & 0xffff), x3 = h2f(v.y >> 16);
#pragma unroll
        for (int g = 0; g < GP; ++g) {
          const float p = sbuf[g * 64 + t];
          a[g][0] = fmaf(p, x0, a[g][0]);
          a[g][1] = fmaf(p, x1, a[g][1]);
          a[g][2] = fmaf(p, x2, a[g][2]);
          a[g][3] = fmaf(p, x3, a[g][3]);
        }
      }
      __syncwarp();
#pragma unroll
      for (int g = 0; g < GP; ++g) *(float4*)(vtmp + g * kD + 4 * lane) = make_float4(a[g][0], a[g][1], a[g][2], a[g][3]);
      add_vtmp();
    }
    F.refill(L, 0, NB, rg, 2 * nk, 2 * k + 1, F.tail_after(2 * k + 1), lane);
  }
  if (cur_u >= 0) flush(cur_u);
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
  int NB, NI, grid, maxseg, G;
  int64_t total;
};

AttnPlan attn_plan(const pkv_layer_t* L, int nblocks, int G) {
  AttnPlan p;
  p.G = G;
  p.NB = max(0, nblocks);
  p.NI = p.NB + res_items(L->buffer);
  const int64_t U = int64_t(L->batch) * L->heads;
  p.total = U * p.NI;
  const int cap = G <= 4 ? attn_grid_cap(attn_fused_kernel<1>) : attn_grid_cap(attn_fused_kernel<2>);
  const int64_t want = (p.total + kWA - 1) / kWA;
  p.grid = int(want < 1 ? 1 : (want < cap ? want : cap));
  const int64_t nwarps = int64_t(p.grid) * kWA;
  // slots per unit: the most warps whose ranges can meet one unit
  const int64_t len_min = p.total / nwarps;
  p.maxseg = len_min == 0 ? int(p.NI < nwarps ? p.NI : nwarps) + 1 : int((p.NI + len_min - 1) / len_min + 1);
  return p;
}

}  // namespace

// Scratch: the arrival counters [U] (zeroed by every call), then the partials
// [U][maxseg][G][kPartA] f32.
int64_t pkv_fast_attention1_scratch(const pkv_layer_t* L, int nblocks, int G) {
  const AttnPlan p = attn_plan(L, nblocks, G);
  const int64_t U = int64_t(L->batch) * L->heads;
  return (U + 3) / 4 * 16 + U * p.maxseg * G * kPartA * 4;
}

int pkv_fast_attention1(const pkv_layer_t* L, int nblocks, const float* q, int G, float* out, void* scratch,
                        cudaStream_t s) {
  const AttnPlan p = attn_plan(L, nblocks, G);
  const int64_t U = int64_t(L->batch) * L->heads;
  int* cnt = (int*)scratch;
  float* part = (float*)((uint8_t*)scratch + (U + 3) / 4 * 16);
  cudaError_t e = cudaMemsetAsync(cnt, 0, U * sizeof(int), s);
  if (e != cudaSuccess) return pkv_cuda_status(e, "pkv_attention_decode(single pass): counters");
  if (G <= 4)
    attn_fused_kernel<1><<<p.grid, kWA * 32, a_smem_bytes(), s>>>(*L, q, G, p.NB, p.NI, p.total, part, p.maxseg, cnt,
                                                                  out);
  else
    attn_fused_kernel<2><<<p.grid, kWA * 32, a_smem_bytes(), s>>>(*L, q, G, p.NB, p.NI, p.total, part, p.maxseg, cnt,
                                                                  out);
  return pkv_cuda_status(cudaGetLastError(), "pkv_attention_decode(single pass)");
}
