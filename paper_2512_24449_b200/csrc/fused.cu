// fused.cu — fused decompress + GEMV over the compressed store
// (SPEC.md:446-463), generic over pack size and head_dim.
//
// One launch covers every (sequence, kv-head) unit, all its blocks and its
// uncompressed residue (single-launch design).  Work unit: a
// warp owns one 64-token block at a time; the block's bytes are staged in the
// warp's shared-memory slot with 16-byte loads (blocks sit at 16-byte-aligned
// arena offsets), the width/minimum header is parsed per lane, payload offsets
// come from a warp prefix scan over the pack widths, and packs
// are decoded in registers and consumed immediately — the decompressed block
// never exists anywhere.  All G query heads of a KV head share
// each decoded pack (GQA).
//
// Lane l owns physical packs l, l+32, ... of every row-group: for the K layout
// (stride-4 interleave) that is 4 adjacent channels 4l..4l+3 at
// head_dim 128, for the V layout channels l, l+32, l+64, l+96.
//
// Dequantisation is factored: sum_c (code*s + z)*q_c = s*sum_c code*q_c +
// z*sum_c q_c (K) and sum_t w_t*(code*s_t + z_t) = sum_t (w_t*s_t)*code +
// sum_t w_t*z_t (V), f32 accumulation; the V reduction across CTAs is a fixed
// order second pass (no atomics; bit-identical run to run).
#include "pkv_common.cuh"

using namespace pkv;

// int8 tensor-core path for the default format (fused_fast.cu)
bool pkv_fast_supported(const pkv_layer_t* L, int G, int64_t stride);
int pkv_fast_fused_k(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
                     cudaStream_t s);
int pkv_fast_fused_v(const pkv_layer_t* L, int nblocks, const float* w, int G, int64_t wstride, float* out,
                     float* part, cudaStream_t s);
int64_t pkv_fast_v_scratch(const pkv_layer_t* L, int nblocks, int G);
int64_t pkv_fast_attention_scratch(const pkv_layer_t* L, int nblocks, int G);
int pkv_fast_attention(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
                       float* out, float* scratch, cudaStream_t s);
// single-pass attention (attn_fused.cu)
int64_t pkv_fast_attention1_scratch(const pkv_layer_t* L, int nblocks, int G);
int pkv_fast_attention1(const pkv_layer_t* L, int nblocks, const float* q, int G, float* out, void* scratch,
                        cudaStream_t s);

namespace {

constexpr int kNW = 4;  // warps per CTA

template <int KP, int D>
struct Cfg {
  static constexpr int ROWS = 64;
  static constexpr int GR = ROWS / KP;
  static constexpr int P = GR * D;
  static constexpr int VPT = D / 32;
  static constexpr int NIB = 8;
  static constexpr int MIN = 8 + (P + 1) / 2;
  static constexpr int PAR = MIN + 2 * P;
  static constexpr int HDR = PAR + 4 * ROWS;
  static constexpr int MAXB = HDR + P * ((KP * 15 + 7) / 8);
  static constexpr int SLOT = ((MAXB + 15) / 16) * 16 + 16;
};

__device__ __forceinline__ void load_block(uint8_t* slot, const uint8_t* src, int len, int lane) {
  const int n16 = (len + 15) >> 4;
  const uint4* s4 = (const uint4*)src;
  uint4* d4 = (uint4*)slot;
  for (int i = lane; i < n16; i += 32) d4[i] = __ldg(s4 + i);
  __syncwarp();
}

__device__ __forceinline__ float h2f(uint16_t v) { return __half2float(__ushort_as_half(v)); }
__device__ __forceinline__ uint16_t sld16(const uint8_t* p) { return *(const uint16_t*)p; }  // 2-aligned

// Per row-group header parse: width, minimum and payload byte offset of the
// lane's VPT packs; `base` advances over the row-group's payloads.
template <int KP, int D>
__device__ __forceinline__ void parse_rowgroup(const uint8_t* slot, int g, int lane, int& base, int (&w)[D / 32],
                                               uint32_t (&mn)[D / 32], int (&off)[D / 32]) {
  using C = Cfg<KP, D>;
#pragma unroll
  for (int i = 0; i < C::VPT; ++i) {
    const int p = g * D + i * 32 + lane;
    const int wi = (slot[C::NIB + (p >> 1)] >> ((p & 1) * 4)) & 15;
    const int pb = (KP * wi + 7) >> 3;
    int inc = pb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(PKV_FULL, inc, o);
      if (lane >= o) inc += y;
    }
    w[i] = wi;
    mn[i] = sld16(slot + C::MIN + 2 * p);
    off[i] = base + inc - pb;
    base += __shfl_sync(PKV_FULL, inc, 31);
  }
}

// ----------------------------------------------------------------- K
template <int KP, int D>
__global__ void __launch_bounds__(kNW * 32) fused_k_kernel(pkv_layer_t L, const float* __restrict__ q, int G,
                                                            float* __restrict__ scores, int64_t sstride, int bpc) {
  using C = Cfg<KP, D>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int u = blockIdx.y, b = u / L.heads, h = u % L.heads, U = L.batch * L.heads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Hq = L.heads * G;
  float* sq = (float*)smem;  // [G][D]
  float* sqsum = sq + G * D; // [G]
  uint8_t* slot = smem + ((G * D + G) * 4 + 15) / 16 * 16 + warp * C::SLOT;
  const float* qu = q + (int64_t(b) * Hq + int64_t(h) * G) * D;
  for (int e = threadIdx.x; e < G * D; e += blockDim.x) sq[e] = qu[e];
  __syncthreads();
  for (int gq = warp; gq < G; gq += kNW) {
    float s = 0.f;
    for (int c = lane; c < D; c += 32) s += sq[gq * D + c];
    s = warp_sum(s);
    if (lane == 0) sqsum[gq] = s;
  }
  __syncthreads();
  const int nb = L.nblk[b];
  const int j0 = blockIdx.x * bpc, j1 = min(nb, j0 + bpc);
  int col[C::VPT];
#pragma unroll
  for (int i = 0; i < C::VPT; ++i) col[i] = kpos_to_col(i * 32 + lane, D);
  const int64_t tab = (int64_t(0) * U + u) * L.max_blocks;
  for (int j = j0 + warp; j < j1; j += kNW) {
    const int64_t off = L.blk_off[tab + j];
    load_block(slot, L.arena + off, L.blk_len[tab + j], lane);
    const uint32_t* words = (const uint32_t*)slot;
    int base = C::HDR;
    for (int g = 0; g < C::GR; ++g) {
      int w[C::VPT], po[C::VPT];
      uint32_t mn[C::VPT];
      parse_rowgroup<KP, D>(slot, g, lane, base, w, mn, po);
      for (int gq = 0; gq < G; ++gq) {
        float part[KP];
#pragma unroll
        for (int t = 0; t < KP; ++t) part[t] = 0.f;
#pragma unroll
        for (int i = 0; i < C::VPT; ++i) {
          const float qv = sq[gq * D + col[i]];
          const uint32_t bit0 = uint32_t(po[i]) * 8u;
#pragma unroll
          for (int t = 0; t < KP; ++t) {
            const uint32_t v = read_bits_aligned(words, bit0 + uint32_t(t * w[i]), w[i]);
            part[t] = fmaf(float(mn[i] + v), qv, part[t]);
          }
        }
        reduce_scatter<KP>(part, lane);
        if (rs_writer<KP>(lane)) {
          const int row = g * KP + rs_index<KP>(lane);
          const float s = h2f(sld16(slot + C::PAR + 4 * row));
          const float z = h2f(sld16(slot + C::PAR + 4 * row + 2));
          scores[(int64_t(b) * Hq + h * G + gq) * sstride + int64_t(j) * C::ROWS + row] =
              fmaf(s, part[0], z * sqsum[gq]);
        }
      }
    }
    __syncwarp();
  }
  if (blockIdx.x == 0) {  // uncompressed residue (staged tokens), same launch
    const int nr = res_rows(L, b, sstride);
    const uint16_t* kr = L.stage + (int64_t(0) * U + u) * L.buffer * D;
    for (int t = warp; t < nr; t += kNW) {
      for (int gq = 0; gq < G; ++gq) {
        float acc = 0.f;
        for (int c = lane; c < D; c += 32) acc = fmaf(h2f(kr[int64_t(t) * D + c]), sq[gq * D + c], acc);
        acc = warp_sum(acc);
        if (lane == 0) scores[(int64_t(b) * Hq + h * G + gq) * sstride + int64_t(nb) * C::ROWS + t] = acc;
      }
    }
  }
}

// ----------------------------------------------------------------- V
template <int KP, int D, int GM>
__global__ void __launch_bounds__(kNW * 32) fused_v_kernel(pkv_layer_t L, const float* __restrict__ w, int G,
                                                            int64_t wstride, float* __restrict__ part, int bpc,
                                                            int nsplit) {
  using C = Cfg<KP, D>;
  extern __shared__ __align__(16) uint8_t smem[];
  const int u = blockIdx.y, b = u / L.heads, h = u % L.heads, U = L.batch * L.heads;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Hq = L.heads * G;
  uint8_t* slot = smem + warp * (C::SLOT + GM * C::ROWS * 4);
  float* ws = (float*)(slot + C::SLOT);  // [GM][64]  w_t * s_t of the current block
  float acc[GM][C::VPT];
  float zacc[GM];
#pragma unroll
  for (int gq = 0; gq < GM; ++gq) {
    zacc[gq] = 0.f;
#pragma unroll
    for (int i = 0; i < C::VPT; ++i) acc[gq][i] = 0.f;
  }
  const float* wu = w + (int64_t(b) * Hq + int64_t(h) * G) * wstride;
  const int nb = L.nblk[b];
  const int j0 = blockIdx.x * bpc, j1 = min(nb, j0 + bpc);
  const int64_t tab = (int64_t(1) * U + u) * L.max_blocks;
  for (int j = j0 + warp; j < j1; j += kNW) {
    const int64_t off = L.blk_off[tab + j];
    load_block(slot, L.arena + off, L.blk_len[tab + j], lane);
    for (int r = lane; r < C::ROWS; r += 32) {
      const float s = h2f(sld16(slot + C::PAR + 4 * r));
      const float z = h2f(sld16(slot + C::PAR + 4 * r + 2));
#pragma unroll
      for (int gq = 0; gq < GM; ++gq) {
        if (gq < G) {
          const float wt = wu[int64_t(gq) * wstride + int64_t(j) * C::ROWS + r];
          ws[gq * C::ROWS + r] = wt * s;
          zacc[gq] = fmaf(wt, z, zacc[gq]);
        }
      }
    }
    __syncwarp();
    const uint32_t* words = (const uint32_t*)slot;
    int base = C::HDR;
    for (int g = 0; g < C::GR; ++g) {
      int wd[C::VPT], po[C::VPT];
      uint32_t mn[C::VPT];
      parse_rowgroup<KP, D>(slot, g, lane, base, wd, mn, po);
#pragma unroll
      for (int i = 0; i < C::VPT; ++i) {
        float code[KP];
        const uint32_t bit0 = uint32_t(po[i]) * 8u;
#pragma unroll
        for (int t = 0; t < KP; ++t) code[t] = float(mn[i] + read_bits_aligned(words, bit0 + uint32_t(t * wd[i]), wd[i]));
#pragma unroll
        for (int gq = 0; gq < GM; ++gq) {
          if (gq < G) {
            float a = 0.f;
#pragma unroll
            for (int t = 0; t < KP; ++t) a = fmaf(ws[gq * C::ROWS + g * KP + t], code[t], a);
            acc[gq][i] += a;
          }
        }
      }
    }
    __syncwarp();
  }
  if (blockIdx.x == 0) {  // residue, same launch; warps split tokens
    const int nr = res_rows(L, b, wstride);
    const uint16_t* vr = L.stage + (int64_t(1) * U + u) * L.buffer * D;
    for (int t = warp; t < nr; t += kNW) {
#pragma unroll
      for (int i = 0; i < C::VPT; ++i) {
        const float v = h2f(vr[int64_t(t) * D + i * 32 + lane]);
#pragma unroll
        for (int gq = 0; gq < GM; ++gq)
          if (gq < G) acc[gq][i] = fmaf(wu[int64_t(gq) * wstride + int64_t(nb) * C::ROWS + t], v, acc[gq][i]);
      }
    }
  }
  // fixed-order cross-warp reduction through shared memory (reuses the slots)
  __syncthreads();
  float* red = (float*)smem;  // [kNW][GM][D+1]
#pragma unroll
  for (int gq = 0; gq < GM; ++gq) {
    if (gq < G) {
#pragma unroll
      for (int i = 0; i < C::VPT; ++i) {
        // V layout: lane l, slot i -> channel i*32 + l
        red[(warp * GM + gq) * (D + 1) + i * 32 + lane] = acc[gq][i];
      }
      const float z = warp_sum(zacc[gq]);
      if (lane == 0) red[(warp * GM + gq) * (D + 1) + D] = z;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < G * (D + 1); e += blockDim.x) {
    const int gq = e / (D + 1), c = e % (D + 1);
    float s = 0.f;
#pragma unroll
    for (int wv = 0; wv < kNW; ++wv) s += red[(wv * GM + gq) * (D + 1) + c];
    part[((int64_t(u) * nsplit + blockIdx.x) * G + gq) * (D + 1) + c] = s;
  }
}

__global__ void fused_v_finalize(const float* __restrict__ part, int U, int heads, int G, int D, int nsplit,
                                 float* __restrict__ out) {
  // out[b][h*G+gq][c], (b*heads + h) = u
  const int64_t total = int64_t(U) * G * D;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int c = int(e % D);
    const int64_t ug = e / D;  // u*G + gq
    const int gq = int(ug % G);
    const int64_t u = ug / G;
    float s = 0.f, z = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float* pp = part + ((u * nsplit + sp) * G + gq) * (D + 1);
      s += pp[c];
      z += pp[D];
    }
    out[e] = s + z;  // [B][Hq][D] with hq = h*G + gq  ==  [(b*heads+h)*G + gq][D]
  }
}

constexpr int kBpc = 16;  // blocks per CTA

template <int KP, int D>
size_t k_smem(int G) {
  return size_t((G * D + G) * 4 + 15) / 16 * 16 + size_t(kNW) * Cfg<KP, D>::SLOT;
}
template <int KP, int D, int GM>
size_t v_smem() {
  const size_t slots = size_t(kNW) * (Cfg<KP, D>::SLOT + GM * 64 * 4);
  const size_t red = size_t(kNW) * GM * (D + 1) * 4;
  return slots > red ? slots : red;
}

template <int KP, int D>
int launch_k(const pkv_layer_t* L, int nblocks, const float* q, int G, float* scores, int64_t sstride,
             cudaStream_t s) {
  const size_t smem = k_smem<KP, D>(G);
  if (smem > 227 * 1024) { pkv_set_error("pack %d / head_dim %d / G %d exceeds shared memory", KP, D, G); return PKV_E_ARG; }
  cudaFuncSetAttribute(fused_k_kernel<KP, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  dim3 grid(max(1, (nblocks + kBpc - 1) / kBpc), L->batch * L->heads);
  fused_k_kernel<KP, D><<<grid, kNW * 32, smem, s>>>(*L, q, G, scores, sstride, kBpc);
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_k_scores");
}

template <int KP, int D, int GM>
int launch_v(const pkv_layer_t* L, int nblocks, const float* w, int G, int64_t wstride, float* out, float* part,
             cudaStream_t s) {
  const size_t smem = v_smem<KP, D, GM>();
  if (smem > 227 * 1024) { pkv_set_error("pack %d / head_dim %d exceeds shared memory", KP, D); return PKV_E_ARG; }
  cudaFuncSetAttribute(fused_v_kernel<KP, D, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  dim3 grid(nsplit, L->batch * L->heads);
  fused_v_kernel<KP, D, GM><<<grid, kNW * 32, smem, s>>>(*L, w, G, wstride, part, kBpc, nsplit);
  const int64_t total = int64_t(L->batch) * L->heads * G * D;
  const int fgrid = int((total + 255) / 256 < 148 * 8 ? (total + 255) / 256 : 148 * 8);
  fused_v_finalize<<<fgrid, 256, 0, s>>>(part, L->batch * L->heads,
                                                                                   L->heads, G, D, nsplit, out);
  return pkv_cuda_status(cudaGetLastError(), "pkv_fused_v_output");
}

int fused_args(const pkv_layer_t* L, int nblocks, int q_heads, int* G) {
  if (!L) { pkv_set_error("null layer"); return PKV_E_ARG; }
  if (L->block != 64) { pkv_set_error("fused kernels need block = 64"); return PKV_E_ARG; }
  if (!(L->head_dim == 64 || L->head_dim == 128 || L->head_dim == 256)) {
    pkv_set_error("fused kernels support head_dim 64/128/256 (got %d)", L->head_dim);
    return PKV_E_ARG;
  }
  if (q_heads <= 0 || q_heads % L->heads) {
    pkv_set_error("q_heads (%d) must be a positive multiple of kv heads (%d)", q_heads, L->heads);
    return PKV_E_SHAPE;
  }
  *G = q_heads / L->heads;
  if (*G > 16) { pkv_set_error("at most 16 query heads per kv head"); return PKV_E_ARG; }
  if (nblocks < 0 || nblocks > L->max_blocks) { pkv_set_error("bad nblocks"); return PKV_E_ARG; }
  return PKV_OK;
}

}  // namespace

#define PKV_DISPATCH_KD(KP_, D_, CALL)                                                    \
  switch (KP_) {                                                                          \
    case 2: { constexpr int KPc = 2; PKV_DISPATCH_D(D_, CALL); } break;                    \
    case 4: { constexpr int KPc = 4; PKV_DISPATCH_D(D_, CALL); } break;                    \
    case 8: { constexpr int KPc = 8; PKV_DISPATCH_D(D_, CALL); } break;                    \
    case 16: { constexpr int KPc = 16; PKV_DISPATCH_D(D_, CALL); } break;                  \
    case 32: { constexpr int KPc = 32; PKV_DISPATCH_D(D_, CALL); } break;                  \
    default: pkv_set_error("bad pack size"); return PKV_E_ARG;                            \
  }
#define PKV_DISPATCH_D(D_, CALL)                                                          \
  switch (D_) {                                                                           \
    case 64: { constexpr int Dc = 64; CALL; } break;                                       \
    case 128: { constexpr int Dc = 128; CALL; } break;                                     \
    case 256: { constexpr int Dc = 256; CALL; } break;                                     \
    default: pkv_set_error("bad head_dim"); return PKV_E_ARG;                             \
  }

extern "C" int pkv_fused_k_scores(const pkv_layer_t* L, int32_t nblocks, const float* q, int32_t q_heads,
                                  float* scores, int64_t score_stride, void* stream) {
  int G = 0;
  int s = fused_args(L, nblocks, q_heads, &G);
  if (s) return s;
  if (score_stride < int64_t(nblocks) * L->block) {
    pkv_set_error("score_stride %lld < nblocks * block = %lld", (long long)score_stride,
                  (long long)nblocks * L->block);
    return PKV_E_SHAPE;
  }
  cudaStream_t strm = (cudaStream_t)stream;
  if (pkv_fast_supported(L, G, score_stride) && (reinterpret_cast<uintptr_t>(q) & 15) == 0) {
    pkv_note_path(PKV_PATH_FAST);
    return pkv_fast_fused_k(L, nblocks, q, G, scores, score_stride, strm);
  }
  pkv_note_path(PKV_PATH_GENERIC);
  PKV_DISPATCH_KD(L->pack_size, L->head_dim, return (launch_k<KPc, Dc>(L, nblocks, q, G, scores, score_stride, strm)));
  return PKV_OK;
}

extern "C" int64_t pkv_fused_v_scratch_bytes(const pkv_layer_t* L, int32_t nblocks, int32_t q_heads) {
  int G = 0;
  if (fused_args(L, nblocks, q_heads, &G)) return -1;
  const int nsplit = max(1, (nblocks + kBpc - 1) / kBpc);
  const int64_t v1 = int64_t(L->batch) * L->heads * nsplit * G * (L->head_dim + 1) * 4;
  const int64_t i8 = pkv_fast_supported(L, G, 4) ? pkv_fast_v_scratch(L, nblocks, G) : 0;
  return v1 > i8 ? v1 : i8;
}

extern "C" int pkv_fused_v_output(const pkv_layer_t* L, int32_t nblocks, const float* w, int32_t q_heads,
                                  int64_t w_stride, float* out, void* scratch, int64_t scratch_bytes,
                                  void* stream) {
  int G = 0;
  int s = fused_args(L, nblocks, q_heads, &G);
  if (s) return s;
  if (scratch_bytes < pkv_fused_v_scratch_bytes(L, nblocks, q_heads)) {
    pkv_set_error("V scratch too small");
    return PKV_E_ARG;
  }
  if (w_stride < int64_t(nblocks) * L->block) {
    pkv_set_error("w_stride %lld < nblocks * block = %lld", (long long)w_stride, (long long)nblocks * L->block);
    return PKV_E_SHAPE;
  }
  cudaStream_t strm = (cudaStream_t)stream;
  float* part = (float*)scratch;
  if (pkv_fast_supported(L, G, w_stride)) {
    pkv_note_path(PKV_PATH_FAST);
    return pkv_fast_fused_v(L, nblocks, w, G, w_stride, out, part, strm);
  }
  pkv_note_path(PKV_PATH_GENERIC);
  if (G <= 4) {
    PKV_DISPATCH_KD(L->pack_size, L->head_dim,
                    return (launch_v<KPc, Dc, 4>(L, nblocks, w, G, w_stride, out, part, strm)));
  } else {
    PKV_DISPATCH_KD(L->pack_size, L->head_dim,
                    return (launch_v<KPc, Dc, 16>(L, nblocks, w, G, w_stride, out, part, strm)));
  }
  return PKV_OK;
}

extern "C" int64_t pkv_attention_scratch_bytes(const pkv_layer_t* L, int32_t nblocks, int32_t q_heads) {
  int G = 0;
  if (fused_args(L, nblocks, q_heads, &G)) return -1;
  if (!pkv_fast_supported(L, G, 4)) return 0;
  // the three-launch path uses the bytes after the single pass's 16-byte work counter
  const int64_t a3 = 16 + pkv_fast_attention_scratch(L, nblocks, G), a1 = pkv_fast_attention1_scratch(L, nblocks, G);
  return a3 > a1 ? a3 : a1;
}

extern "C" int pkv_attention_decode(const pkv_layer_t* L, int32_t nblocks, const float* q, int32_t q_heads,
                                    float* scores, int64_t score_stride, float* out, void* scratch,
                                    int64_t scratch_bytes, void* stream) {
  int G = 0;
  int s = fused_args(L, nblocks, q_heads, &G);
  if (s) return s;
  if (!pkv_fast_supported(L, G, score_stride) || (reinterpret_cast<uintptr_t>(q) & 15) ||
      (reinterpret_cast<uintptr_t>(out) & 15)) {
    pkv_set_error("attention_decode: only the default format (pack 16, head_dim 128, block 64, G <= 8) is fused");
    return PKV_E_ARG;
  }
  if (!scores) {  // single pass: no score rows
    if (scratch_bytes < pkv_fast_attention1_scratch(L, nblocks, G) || (reinterpret_cast<uintptr_t>(scratch) & 15)) {
      pkv_set_error("attention scratch too small or misaligned");
      return PKV_E_ARG;
    }
    pkv_note_path(PKV_PATH_SINGLE);
    return pkv_fast_attention1(L, nblocks, q, G, out, scratch, (cudaStream_t)stream);
  }
  if (score_stride < int64_t(nblocks) * L->block) {
    pkv_set_error("score_stride %lld < nblocks * block = %lld", (long long)score_stride,
                  (long long)nblocks * L->block);
    return PKV_E_SHAPE;
  }
  if (scratch_bytes < 16 + pkv_fast_attention_scratch(L, nblocks, G)) {
    pkv_set_error("attention scratch too small");
    return PKV_E_ARG;
  }
  pkv_note_path(PKV_PATH_FAST);
  return pkv_fast_attention(L, nblocks, q, G, scores, score_stride, out, (float*)((uint8_t*)scratch + 16),
                            (cudaStream_t)stream);
}
