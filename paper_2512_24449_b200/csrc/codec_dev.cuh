// codec_dev.cuh — device building blocks shared by codec.cu and store.cu.
#pragma once
#include "pkv_common.cuh"

namespace pkv {

// ---- quantize one row with a warp ----
// f32 arithmetic with explicit round-to-nearest intrinsics (no contraction),
// IEEE divide, round-half-away-from-zero via roundf; codes >= 2^16 flag a width
// overflow (the oracle raises WidthOverflowError at encode time for them).
__device__ __forceinline__ void quantize_row_warp(const uint16_t* __restrict__ src, int cols, float rel,
                                                  uint16_t* __restrict__ q, float* __restrict__ params,
                                                  int32_t* err, int lane) {
  float mn = __int_as_float(0x7f800000), mx = -__int_as_float(0x7f800000);
  bool bad = false;
  for (int c = lane; c < cols; c += 32) {
    const float x = __half2float(__ushort_as_half(src[c]));
    bad |= !isfinite(x);
    mn = fminf(mn, x);
    mx = fmaxf(mx, x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(PKV_FULL, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(PKV_FULL, mx, o));
  }
  bad = __any_sync(PKV_FULL, bad);
  if (bad && lane == 0) set_flag(err, PKV_FLAG_NONFINITE);
  const float scale = __fmul_rn(rel, __fsub_rn(mx, mn));
  bool wide = false;
  for (int c = lane; c < cols; c += 32) {
    const float x = __half2float(__ushort_as_half(src[c]));
    float r = 0.f;
    if (scale > 0.f) r = roundf(__fdiv_rn(__fsub_rn(x, mn), scale));
    if (!(r <= 65535.f)) { wide = true; r = 65535.f; }
    q[c] = uint16_t(r);
  }
  if (__any_sync(PKV_FULL, wide) && lane == 0) set_flag(err, PKV_FLAG_WIDTH);
  if (lane == 0) {
    params[0] = scale;
    params[1] = mn;
  }
}

// ---- encode ----
struct EncSrc {
  const uint16_t* codes;  // [rows][cols] source rows
  const uint8_t* perm;    // block row -> source row (nullptr = identity)
  const float* params;    // [rows][2] (scale, zp) by source row (nullptr = zeros)
};

__device__ __forceinline__ int src_row(const EncSrc& s, int r) { return s.perm ? int(s.perm[r]) : r; }

__host__ __device__ inline size_t round16s(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline size_t size_smem_bytes(const Fmt& f) {
  return round16s(f.P) + round16s(2 * size_t(f.P)) + 4 * size_t(f.P) + 64;
}
__host__ __device__ inline size_t enc_smem_bytes(const Fmt& f) {
  return size_smem_bytes(f) + round16s(max_block_bytes(f)) + 16;
}

// In-place exclusive scan of arr[0..n) by the whole CTA (blockDim.x a multiple
// of 32, <= 1024).  Returns the total on every thread.  `scratch` holds
// >= blockDim.x / 32 + 1 ints.
__device__ inline int32_t cta_exclusive_scan(int32_t* arr, int n, int32_t* scratch) {
  const int t = threadIdx.x, nt = blockDim.x;
  const int chunk = (n + nt - 1) / nt;
  const int b0 = min(n, t * chunk), b1 = min(n, b0 + chunk);
  int32_t s = 0;
  for (int i = b0; i < b1; ++i) s += arr[i];
  // warp inclusive scan
  const int lane = t & 31, wid = t >> 5;
  int32_t inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(PKV_FULL, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) scratch[wid] = inc;
  __syncthreads();
  if (t == 0) {
    int32_t acc = 0;
    for (int w = 0; w < nt / 32; ++w) {
      const int32_t v = scratch[w];
      scratch[w] = acc;
      acc += v;
    }
    scratch[nt / 32] = acc;
  }
  __syncthreads();
  int32_t run = scratch[wid] + inc - s;
  for (int i = b0; i < b1; ++i) {
    const int32_t v = arr[i];
    arr[i] = run;
    run += v;
  }
  const int32_t total = scratch[nt / 32];
  __syncthreads();
  return total;
}

// Computes widths, minima and payload offsets of every pack into shared
// memory (sw / smn / soff) and returns the exact block byte length.
__device__ inline int64_t block_layout_dev(const EncSrc& src, const Fmt& f, int layout, uint8_t* smem,
                                           int32_t* err) {
  uint8_t* sw = smem;
  uint16_t* smn = (uint16_t*)(smem + round16s(f.P));
  int32_t* soff = (int32_t*)(smem + round16s(f.P) + round16s(2 * size_t(f.P)));
  int32_t* sscan = soff + f.P;
  bool wide = false;
  for (int p = threadIdx.x; p < f.P; p += blockDim.x) {
    const int g = p / f.cols, pos = p - g * f.cols;
    const int c = pos_to_col(pos, f.cols, layout);
    uint32_t lo = 0xffffffffu, hi = 0;
    for (int j = 0; j < f.k; ++j) {
      const uint32_t v = src.codes[int64_t(src_row(src, g * f.k + j)) * f.cols + c];
      lo = min(lo, v);
      hi = max(hi, v);
    }
    int w = width_of(hi - lo);
    if (w > 15) { wide = true; w = 15; }
    sw[p] = uint8_t(w);
    smn[p] = uint16_t(lo);
    soff[p] = (f.k * w + 7) >> 3;
  }
  if (__syncthreads_or(wide) && threadIdx.x == 0) set_flag(err, PKV_FLAG_WIDTH);
  const int32_t pay = cta_exclusive_scan(soff, f.P, sscan);
  return int64_t(f.hdr) + pay;
}

// Encodes one block (whole CTA) into `dst`.  pad16: dst is 16-byte aligned and
// owns round16(len) bytes (zero padding written); otherwise exactly len bytes.
__device__ inline int64_t encode_block_dev(const EncSrc& src, const Fmt& f, int layout, int kind,
                                           uint8_t* smem, uint8_t* dst, bool pad16, int32_t* err) {
  const int64_t total = block_layout_dev(src, f, layout, smem, err);
  uint8_t* sw = smem;
  uint16_t* smn = (uint16_t*)(smem + round16s(f.P));
  int32_t* soff = (int32_t*)(smem + round16s(f.P) + round16s(2 * size_t(f.P)));
  uint8_t* sbuf = smem + size_smem_bytes(f);
  const int t = threadIdx.x, nt = blockDim.x;
  const int64_t padded = round16(total);
  for (int64_t i = total + t; i < padded; i += nt) sbuf[i] = 0;
  if (t == 0) {
    sbuf[0] = uint8_t(kind);
    sbuf[1] = uint8_t(layout);
    sbuf[2] = uint8_t(f.k);
    sbuf[3] = 0;
    sbuf[4] = uint8_t(f.rows & 0xff);
    sbuf[5] = uint8_t(f.rows >> 8);
    sbuf[6] = uint8_t(f.cols & 0xff);
    sbuf[7] = uint8_t(f.cols >> 8);
  }
  for (int b = t; b < (f.P + 1) / 2; b += nt) {
    const int p = 2 * b;
    const uint8_t lo = sw[p], hi = (p + 1 < f.P) ? sw[p + 1] : 0;
    sbuf[f.nib_off + b] = uint8_t(lo | (hi << 4));
  }
  for (int p = t; p < f.P; p += nt) {
    sbuf[f.min_off + 2 * p] = uint8_t(smn[p] & 0xff);
    sbuf[f.min_off + 2 * p + 1] = uint8_t(smn[p] >> 8);
  }
  bool ovf = false;
  for (int r = t; r < f.rows; r += nt) {
    float s = 0.f, z = 0.f;
    if (src.params) {
      const int sr = src_row(src, r);
      s = src.params[2 * sr];
      z = src.params[2 * sr + 1];
    }
    // Move the f16 bit patterns through a 32-bit integer register: without the
    // asm barrier ptxas folds "cvt.f16 then st.u8" into a numeric F2I.U8.
    uint32_t s16 = __half_as_ushort(__float2half_rn(s));
    uint32_t z16 = __half_as_ushort(__float2half_rn(z));
    asm volatile("" : "+r"(s16), "+r"(z16));
    if ((s16 & 0x7c00) == 0x7c00) ovf = true;  // scale not representable in f16
    uint8_t* pp = sbuf + f.par_off + 4 * r;
    pp[0] = uint8_t(s16 & 0xff);
    pp[1] = uint8_t(s16 >> 8);
    pp[2] = uint8_t(z16 & 0xff);
    pp[3] = uint8_t(z16 >> 8);
  }
  if (ovf) set_flag(err, PKV_FLAG_WIDTH);
  for (int p = t; p < f.P; p += nt) {
    const int w = sw[p];
    if (w == 0) continue;
    const int g = p / f.cols, pos = p - g * f.cols;
    const int c = pos_to_col(pos, f.cols, layout);
    const uint32_t mn = smn[p];
    uint8_t* o = sbuf + f.hdr + soff[p];
    uint64_t acc = 0;
    int nbits = 0, ob = 0;
    for (int j = 0; j < f.k; ++j) {
      const uint32_t v = src.codes[int64_t(src_row(src, g * f.k + j)) * f.cols + c] - mn;
      acc |= uint64_t(v & ((1u << w) - 1u)) << nbits;
      nbits += w;
      while (nbits >= 8) {
        o[ob++] = uint8_t(acc & 0xff);
        acc >>= 8;
        nbits -= 8;
      }
    }
    if (nbits > 0) o[ob++] = uint8_t(acc & 0xff);
  }
  __syncthreads();
  if (pad16) {
    const uint4* s4 = (const uint4*)sbuf;
    uint4* d4 = (uint4*)dst;
    for (int64_t i = t; i < padded / 16; i += nt) d4[i] = s4[i];
  } else {
    for (int64_t i = t; i < total; i += nt) dst[i] = sbuf[i];
  }
  __syncthreads();
  return total;
}

// ---- decode ----
__device__ __forceinline__ uint32_t read_bits_bytes(const uint8_t* p, int bit, int w) {
  if (w == 0) return 0;
  const uint8_t* b = p + (bit >> 3);
  const int sh = bit & 7;
  const int nb = (sh + w + 7) >> 3;
  uint32_t v = 0;
  for (int i = 0; i < nb; ++i) v |= uint32_t(b[i]) << (8 * i);
  return (v >> sh) & ((1u << w) - 1u);
}

__device__ __forceinline__ bool valid_pack_size(int k) {
  return k == 2 || k == 4 || k == 8 || k == 16 || k == 32;
}

// Decodes one block (whole CTA); validates header and length (MalformedBlockError).
__device__ inline void decode_block_dev(const uint8_t* __restrict__ b, int64_t len, int rows_exp, int cols_exp,
                                        uint16_t* __restrict__ q, float* __restrict__ params, int32_t* scratch,
                                        int32_t* err) {
  bool ok = len >= 8;
  int kind = 0, layout = 0, k = 16, rows = 0, cols = 0;
  if (ok) {
    kind = b[0];
    layout = b[1];
    k = b[2];
    rows = ld16le(b + 4);
    cols = ld16le(b + 6);
    ok = kind <= 1 && layout <= 1 && valid_pack_size(k) && rows == rows_exp && cols == cols_exp &&
         rows % k == 0;
  }
  Fmt f = make_fmt(ok ? rows : 0, ok ? cols : 0, ok ? k : 16);
  ok = ok && len >= f.hdr;
  if (!ok) {
    if (threadIdx.x == 0) set_flag(err, PKV_FLAG_MALFORMED);
    return;
  }
  int32_t* soff = scratch;
  int32_t* sscan = scratch + f.P;
  for (int p = threadIdx.x; p < f.P; p += blockDim.x) {
    const int w = (b[f.nib_off + (p >> 1)] >> ((p & 1) * 4)) & 15;
    soff[p] = (k * w + 7) >> 3;
  }
  __syncthreads();
  const int32_t pay = cta_exclusive_scan(soff, f.P, sscan);
  if (int64_t(f.hdr) + pay != len) {
    if (threadIdx.x == 0) set_flag(err, PKV_FLAG_MALFORMED);
    return;
  }
  for (int p = threadIdx.x; p < f.P; p += blockDim.x) {
    const int w = (b[f.nib_off + (p >> 1)] >> ((p & 1) * 4)) & 15;
    const uint32_t mn = ld16le(b + f.min_off + 2 * p);
    const int g = p / f.cols, pos = p - g * f.cols;
    const int c = pos_to_col(pos, f.cols, layout);
    const uint8_t* pay_p = b + f.hdr + soff[p];
    for (int j = 0; j < k; ++j)
      q[int64_t(g * k + j) * f.cols + c] = uint16_t(mn + read_bits_bytes(pay_p, j * w, w));
  }
  for (int r = threadIdx.x; r < f.rows; r += blockDim.x) {
    params[2 * r] = __half2float(__ushort_as_half(ld16le(b + f.par_off + 4 * r)));
    params[2 * r + 1] = __half2float(__ushort_as_half(ld16le(b + f.par_off + 4 * r + 2)));
  }
}

}  // namespace pkv
