// codec.cu — quantizer and bit-pack codec kernels (generic rows/cols/pack size).
//
//  quantize_row     SPEC.md:111-119  (f32, IEEE divide, round-half-away)
//  dequantize       SPEC.md:120-128  (q*scale + zp, mul then add)
//  encode_block     SPEC.md:275-283, wire layout SPEC.md:330
//  decode_block
//  decode_pack_at
//
// These generic kernels serve the API-level codec calls and the store's flush
// pipeline (store.cu); the decode-time hot path lives in fused.cu.
#include "codec_dev.cuh"

using namespace pkv;

namespace {

constexpr int kThreads = 256;

__global__ void quantize_kernel(const uint16_t* __restrict__ x, int nrows_total, int cols, float rel,
                                uint16_t* __restrict__ q, float* __restrict__ params, int32_t* err) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nrows_total) return;
  const uint16_t* src = x + int64_t(warp) * cols;
  quantize_row_warp(src, cols, rel, q + int64_t(warp) * cols, params + 2 * int64_t(warp), err, lane);
}

__global__ void check_finite_kernel(const uint16_t* __restrict__ x, int64_t n, int32_t* err) {
  bool bad = false;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    bad |= (x[i] & 0x7c00) == 0x7c00;  // exponent all ones: inf or nan
  if (__syncthreads_or(bad) && threadIdx.x == 0) set_flag(err, PKV_FLAG_NONFINITE);
}

__global__ void dequantize_kernel(const uint16_t* __restrict__ q, const float* __restrict__ params,
                                  int64_t total, int cols, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i / cols;
    const float s = params[2 * row], z = params[2 * row + 1];
    out[i] = __fadd_rn(__fmul_rn(float(q[i]), s), z);
  }
}

__global__ void encode_sizes_kernel(const uint16_t* __restrict__ q, int rows, int cols, int k, int layout,
                                    int64_t* sizes, int32_t* err) {
  extern __shared__ __align__(16) uint8_t smem[];
  const Fmt f = make_fmt(rows, cols, k);
  EncSrc src{q + int64_t(blockIdx.x) * rows * cols, nullptr, nullptr};
  const int64_t total = block_layout_dev(src, f, layout, smem, err);
  if (threadIdx.x == 0) sizes[blockIdx.x] = total;
}

__global__ void encode_kernel(const uint16_t* __restrict__ q, const float* __restrict__ params, int rows,
                              int cols, int k, int layout, int kind, const int64_t* __restrict__ offsets,
                              uint8_t* out, int32_t* err) {
  extern __shared__ __align__(16) uint8_t smem[];
  const Fmt f = make_fmt(rows, cols, k);
  EncSrc src{q + int64_t(blockIdx.x) * rows * cols, nullptr,
             params ? params + int64_t(blockIdx.x) * rows * 2 : nullptr};
  encode_block_dev(src, f, layout, kind, smem, out + offsets[blockIdx.x], /*pad16=*/false, err);
}

__global__ void decode_kernel(const uint8_t* __restrict__ buf, const int64_t* __restrict__ offsets,
                              const int64_t* __restrict__ lens, int rows, int cols, uint16_t* q,
                              float* params, int32_t* err) {
  extern __shared__ __align__(16) uint8_t smem[];
  decode_block_dev(buf + offsets[blockIdx.x], lens[blockIdx.x], rows, cols,
                   q + int64_t(blockIdx.x) * rows * cols, params + int64_t(blockIdx.x) * rows * 2,
                   (int32_t*)smem, err);
}

__global__ void decode_pack_at_kernel(const uint8_t* __restrict__ buf, const int64_t* __restrict__ offsets,
                                      int n, int pack, uint16_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint8_t* b = buf + offsets[i];
  const int k = b[2], rows = ld16le(b + 4), cols = ld16le(b + 6);
  const Fmt f = make_fmt(rows, cols, k);
  // payload offset: prefix over widths of the packs before `pack` (one scan)
  int64_t off = f.hdr;
  for (int p = 0; p < pack; ++p) {
    const int w = (b[f.nib_off + (p >> 1)] >> ((p & 1) * 4)) & 15;
    off += (k * w + 7) >> 3;
  }
  const int w = (b[f.nib_off + (pack >> 1)] >> ((pack & 1) * 4)) & 15;
  const uint16_t mn = ld16le(b + f.min_off + 2 * pack);
  for (int j = 0; j < k; ++j) out[int64_t(i) * k + j] = uint16_t(mn + read_bits_bytes(b + off, j * w, w));
}

}  // namespace

static int launch_status(const char* what) { return pkv_cuda_status(cudaGetLastError(), what); }

extern "C" int pkv_quantize(const uint16_t* x, int32_t n, int32_t rows, int32_t cols, float rel, uint16_t* q,
                            float* params, int32_t* err, void* stream) {
  if (n < 0 || rows < 0 || cols < 0) { pkv_set_error("negative shape"); return PKV_E_SHAPE; }
  if (!(rel > 0.f && rel <= 1.f)) { pkv_set_error("rel_quant_scale must be in (0, 1]"); return PKV_E_ARG; }
  const int64_t nrows = int64_t(n) * rows;
  if (nrows == 0 || cols == 0) return PKV_OK;
  const int warps_per_cta = kThreads / 32;
  const int64_t grid = (nrows + warps_per_cta - 1) / warps_per_cta;
  quantize_kernel<<<dim3(unsigned(grid)), kThreads, 0, (cudaStream_t)stream>>>(x, int(nrows), cols, rel, q,
                                                                                params, err);
  return launch_status("pkv_quantize");
}

extern "C" int pkv_check_finite(const uint16_t* x, int64_t n, int32_t* err, void* stream) {
  if (n <= 0) return PKV_OK;
  const int64_t grid = (n + kThreads - 1) / kThreads;
  check_finite_kernel<<<unsigned(grid < 148 * 8 ? grid : 148 * 8), kThreads, 0, (cudaStream_t)stream>>>(x, n, err);
  return launch_status("pkv_check_finite");
}

// dst = scale * src over n f32; either side may be pinned host memory, which
// the SMs read / write over PCIe directly (UVA), so a decode step's query can
// arrive from host memory already prescaled and its output leave to host
// memory inside one CUDA graph, without copy-engine transfers.  float4 when
// both pointers are 16-byte aligned and n % 4 == 0.
__global__ void copy_scaled_kernel(const float* __restrict__ src, float* __restrict__ dst, int64_t n, float scale,
                                   bool vec) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vec) {
    for (; i < n / 4; i += stride) {
      float4 v = reinterpret_cast<const float4*>(src)[i];
      v.x *= scale;
      v.y *= scale;
      v.z *= scale;
      v.w *= scale;
      reinterpret_cast<float4*>(dst)[i] = v;
    }
  } else {
    for (; i < n; i += stride) dst[i] = src[i] * scale;
  }
}

extern "C" int pkv_copy_scaled(const float* src, float* dst, int64_t n, float scale, void* stream) {
  if (n < 0 || (n > 0 && (!src || !dst))) { pkv_set_error("pkv_copy_scaled: bad arguments"); return PKV_E_ARG; }
  if (n == 0) return PKV_OK;
  const bool vec = n % 4 == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  const int64_t items = vec ? n / 4 : n;
  // one element (or float4) per thread up to 148 x 8 CTAs: many small reads in
  // flight is what a PCIe-mapped source needs
  const int64_t grid = (items + kThreads - 1) / kThreads;
  copy_scaled_kernel<<<unsigned(grid < 148 * 8 ? grid : 148 * 8), kThreads, 0, (cudaStream_t)stream>>>(src, dst, n,
                                                                                                   scale, vec);
  return launch_status("pkv_copy_scaled");
}

extern "C" int pkv_dequantize(const uint16_t* q, const float* params, int32_t n, int32_t rows, int32_t cols,
                              float* out, void* stream) {
  const int64_t total = int64_t(n) * rows * cols;
  if (total == 0) return PKV_OK;
  const int64_t grid = (total + kThreads - 1) / kThreads;
  dequantize_kernel<<<unsigned(grid < 148 * 16 ? grid : 148 * 16), kThreads, 0, (cudaStream_t)stream>>>(
      q, params, total, cols, out);
  return launch_status("pkv_dequantize");
}

static int check_codec_args(int32_t rows, int32_t cols, int32_t k, int32_t layout, size_t* smem_enc) {
  if (!(k == 2 || k == 4 || k == 8 || k == 16 || k == 32)) {
    pkv_set_error("pack_size must be one of 2,4,8,16,32");
    return PKV_E_ARG;
  }
  if (layout != 0 && layout != 1) { pkv_set_error("bad layout"); return PKV_E_ARG; }
  if (rows <= 0 || cols <= 0 || rows % k != 0) {
    pkv_set_error("rows (%d) must be a positive multiple of pack_size (%d)", rows, k);
    return PKV_E_SHAPE;
  }
  const Fmt f = make_fmt(rows, cols, k);
  *smem_enc = enc_smem_bytes(f);
  if (*smem_enc > 220 * 1024 || rows > 65535 || cols > 65535) {
    pkv_set_error("block %dx%d (pack %d) exceeds the device codec limit", rows, cols, k);
    return PKV_E_ARG;
  }
  return PKV_OK;
}

extern "C" int pkv_encode_sizes(const uint16_t* q, int32_t n, int32_t rows, int32_t cols, int32_t pack_size,
                                int32_t layout, int64_t* sizes, int32_t* err, void* stream) {
  size_t smem = 0;
  int st = check_codec_args(rows, cols, pack_size, layout, &smem);
  if (st) return st;
  if (n == 0) return PKV_OK;
  const size_t smem_sz = size_smem_bytes(make_fmt(rows, cols, pack_size));
  cudaFuncSetAttribute(encode_sizes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_sz));
  encode_sizes_kernel<<<n, kThreads, smem_sz, (cudaStream_t)stream>>>(q, rows, cols, pack_size, layout, sizes,
                                                                        err);
  return launch_status("pkv_encode_sizes");
}

extern "C" int pkv_encode(const uint16_t* q, const float* params, int32_t n, int32_t rows, int32_t cols,
                          int32_t pack_size, int32_t layout, int32_t kind, const int64_t* offsets, uint8_t* out,
                          int32_t* err, void* stream) {
  size_t smem = 0;
  int st = check_codec_args(rows, cols, pack_size, layout, &smem);
  if (st) return st;
  if (kind != 0 && kind != 1) { pkv_set_error("bad kind"); return PKV_E_ARG; }
  if (n == 0) return PKV_OK;
  cudaFuncSetAttribute(encode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  encode_kernel<<<n, kThreads, smem, (cudaStream_t)stream>>>(q, params, rows, cols, pack_size, layout, kind,
                                                               offsets, out, err);
  return launch_status("pkv_encode");
}

extern "C" int pkv_decode(const uint8_t* buf, const int64_t* offsets, const int64_t* lens, int32_t n,
                          int32_t rows, int32_t cols, uint16_t* q, float* params, int32_t* err, void* stream) {
  if (n == 0) return PKV_OK;
  if (rows <= 0 || cols <= 0 || rows > 65535 || cols > 65535) { pkv_set_error("bad shape"); return PKV_E_SHAPE; }
  // widths+offset scratch for the largest pack count (pack_size 2)
  const size_t smem = size_t(rows / 2) * cols * sizeof(int32_t) + 64;
  if (smem > 220 * 1024) { pkv_set_error("block too large for device decode"); return PKV_E_ARG; }
  cudaFuncSetAttribute(decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  decode_kernel<<<n, kThreads, smem, (cudaStream_t)stream>>>(buf, offsets, lens, rows, cols, q, params, err);
  return launch_status("pkv_decode");
}

extern "C" int pkv_decode_pack_at(const uint8_t* buf, const int64_t* offsets, int32_t n, int32_t pack_index,
                                  uint16_t* out, void* stream) {
  if (n == 0) return PKV_OK;
  decode_pack_at_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(buf, offsets, n, pack_index, out);
  return launch_status("pkv_decode_pack_at");
}
