// pkv_common.cuh — shared definitions for the sm_100a PackKV kernels.
//
// Wire format of one PackedBlock (byte map SURVEY.md Appendix C):
//   [0,8)    kind u8 | layout u8 | pack_size u8 | reserved u8 | rows u16 | cols u16
//   [8, +ceil(P/2))   4-bit widths, physical pack order, even pack in the low nibble
//   [.., +2P)         minima u16 LE, physical order
//   [.., +4*rows)     per-row (scale f16, zp f16)
//   [hdr, ...)        payloads, pack p at hdr + sum_{j<p} ceil(k*w_j/8); value j of a
//                     pack at bits [j*w, (j+1)*w), little-endian bit numbering
// with P = (rows/k)*cols packs; physical pack p = g*cols + pos(c) for row-group g
// and column c; pos(c) = c for the V layout and the stride-4 interleave
// pos(c) = sum_{r < c%4} ceil((cols-r)/4) + c/4 for the K layout.
#pragma once
#include <utility>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/packkv_b200.h"

#define PKV_FULL 0xffffffffu

namespace pkv {

struct Fmt {
  int rows, cols, k, G, P;
  int nib_off, min_off, par_off, hdr;
};

__host__ __device__ inline Fmt make_fmt(int rows, int cols, int k) {
  Fmt f;
  f.rows = rows;
  f.cols = cols;
  f.k = k;
  f.G = rows / k;
  f.P = f.G * cols;
  f.nib_off = 8;
  f.min_off = 8 + (f.P + 1) / 2;
  f.par_off = f.min_off + 2 * f.P;
  f.hdr = f.par_off + 4 * rows;
  return f;
}

__host__ __device__ inline int max_payload(int k) { return (k * 15 + 7) / 8; }
__host__ __device__ inline int max_block_bytes(const Fmt& f) { return f.hdr + f.P * max_payload(f.k); }
__host__ __device__ inline int64_t round16(int64_t x) { return (x + 15) & ~int64_t(15); }

// K layout: physical position -> column and back (general cols).
__host__ __device__ inline int kpos_to_col(int pos, int cols) {
  const int c0 = (cols + 3) / 4, c1 = (cols + 2) / 4, c2 = (cols + 1) / 4;
  if (pos < c0) return 4 * pos;
  if (pos < c0 + c1) return 4 * (pos - c0) + 1;
  if (pos < c0 + c1 + c2) return 4 * (pos - c0 - c1) + 2;
  return 4 * (pos - c0 - c1 - c2) + 3;
}
__host__ __device__ inline int col_to_kpos(int c, int cols) {
  const int r = c & 3;
  int base = 0;
  for (int s = 0; s < r; ++s) base += (cols - s + 3) / 4;
  return base + (c >> 2);
}
__host__ __device__ inline int pos_to_col(int pos, int cols, int layout) {
  return layout == PKV_LAYOUT_K_INTERLEAVED ? kpos_to_col(pos, cols) : pos;
}

__device__ __forceinline__ int width_of(uint32_t range) { return range ? 32 - __clz(range) : 0; }

// Little-endian bitfield read of `w` (<= 25) bits starting at absolute bit
// `bit` of a 4-byte-aligned byte buffer (reads two aligned words).
__device__ __forceinline__ uint32_t read_bits_aligned(const uint32_t* words, uint32_t bit, int w) {
  const uint32_t i = bit >> 5, sh = bit & 31;
  const uint32_t lo = words[i], hi = words[i + 1];
  const uint32_t v = __funnelshift_r(lo, hi, sh);
  return w >= 32 ? v : (v & ((1u << w) - 1u));
}

__device__ __forceinline__ uint8_t ldb(const uint8_t* p) { return *p; }
__device__ __forceinline__ uint16_t ld16le(const uint8_t* p) { return uint16_t(p[0]) | (uint16_t(p[1]) << 8); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(PKV_FULL, v, o);
  return v;
}

// Transpose-reduce K per-lane values across the warp: afterwards v[0] on every
// lane holds the warp-wide sum of index rs_index<K>(lane).  K power of 2 <= 32.
template <int K>
__device__ __forceinline__ void reduce_scatter(float (&v)[K], int lane) {
  int n = K;
  int m = 16;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    if ((K >> s) <= 1) break;
    const int h = (K >> s) / 2;
    const bool up = (lane & m) != 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < h) {
        const float send = up ? v[i] : v[i + h];
        const float keep = up ? v[i + h] : v[i];
        v[i] = keep + __shfl_xor_sync(PKV_FULL, send, m);
      }
    }
    m >>= 1;
    n = h;
  }
  (void)n;
  for (; m > 0; m >>= 1) v[0] += __shfl_xor_sync(PKV_FULL, v[0], m);
}
template <int K>
__device__ __forceinline__ int rs_index(int lane) {
  int idx = 0, m = 16;
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    if ((K >> s) <= 1) break;
    const int h = (K >> s) / 2;
    if (lane & m) idx += h;
    m >>= 1;
  }
  return idx;
}
template <int K>
__device__ __forceinline__ bool rs_writer(int lane) {
  // lanes whose bits below the last used mask are zero
  int used = 0;
  for (int s = 0; s < 5; ++s) {
    if ((K >> s) <= 1) break;
    ++used;
  }
  const int low = 5 - used;
  return (lane & ((1 << low) - 1)) == 0;
}

// Programmatic dependent launch (the decode-step kernels, launched with
// pkv_launch_pdl): the next kernel of the stream may start its prologue while
// this one runs; pdl_wait() blocks until the previous kernel has completed and
// its writes are visible, pdl_launch() lets the next kernel start.  Both are
// no-ops for a kernel launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void set_flag(int32_t* err, int32_t bit) {
  if (err) atomicOr(err, bit);
}

// Residue rows of sequence b that fit a score / weight row of `stride` floats
// (rows nblk*block + t, t < nres).  A caller stride shorter than the token
// count drops the rows past it and raises PKV_FLAG_SHAPE (ShapeMismatchError)
// instead of writing / reading into the next head's row.
__device__ __forceinline__ int res_rows(const pkv_layer_t& L, int b, int64_t stride) {
  const int nr = L.nres[b];
  const int64_t room = stride - int64_t(L.nblk[b]) * L.block;
  if (int64_t(nr) <= room) return nr;
  if (threadIdx.x % 32 == 0) set_flag(L.err, PKV_FLAG_SHAPE);
  return room > 0 ? int(room) : 0;
}

}  // namespace pkv

// host-side helpers (defined in capi.cu)
bool pkv_pdl_enabled();  // PKV_PDL=0 disables programmatic dependent launch
// <<<grid, block, smem, stream>>> with programmatic stream serialization
// allowed (the kernel must call pdl_wait() before reading what the previous
// kernel writes)
template <typename... KArgs, typename... Args>
cudaError_t pkv_launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                           Args&&... args) {
  if (!pkv_pdl_enabled()) {
    kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
void pkv_set_error(const char* fmt, ...);
int pkv_cuda_status(cudaError_t e, const char* what);
void pkv_note_path(int path);  // records the kernel family for pkv_last_path()
