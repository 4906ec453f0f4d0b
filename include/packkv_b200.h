/*
 * packkv_b200.h — C ABI of the B200-native PackKV hot path (libpackkv_b200.so).
 *
 * The reference (arXiv 2512.24449, /root/reference) ships a pure-Python API
 * and no FFI: SPEC.md specifies the functions below as Python operations.
 * Each entry point here replaces one of them (cited per function); the
 * Python package paper_2512_24449_b200 binds them with ctypes exactly as a
 * maintainer would bind them from packkv.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer owned by the caller (the library never
 *     allocates or frees device memory; torch allocates arenas, tables,
 *     scratch and outputs);
 *   - every call is asynchronous on `stream` (a cudaStream_t passed as void*);
 *   - every call returns PKV_OK or a PKV_E_* status; pkv_last_error() gives a
 *     thread-local message.  Data-dependent errors that only the device can
 *     see (non-finite input, width overflow, malformed block) are OR-ed into
 *     the caller's int32 `err` flag word as PKV_FLAG_* bits, to be checked by
 *     the caller after a stream sync (the Python layer maps them onto
 *     packkv.errors classes: NonFiniteValueError, WidthOverflowError,
 *     MalformedBlockError — errors.py:20,28,32).
 *   - fp16 tensors are passed as uint16_t* (raw IEEE binary16 bit patterns).
 */
#ifndef PACKKV_B200_H
#define PACKKV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PKV_ABI_VERSION 1

enum {
  PKV_OK = 0,
  PKV_E_SHAPE = 1,      /* ShapeMismatchError (errors.py:24)          */
  PKV_E_NONFINITE = 2,  /* NonFiniteValueError (errors.py:20)         */
  PKV_E_WIDTH = 3,      /* WidthOverflowError (errors.py:28)          */
  PKV_E_MALFORMED = 4,  /* MalformedBlockError (errors.py:32)         */
  PKV_E_INDEX = 5,      /* IndexError         */
  PKV_E_ARG = 6,        /* ValueError: unsupported parameter          */
  PKV_E_CUDA = 7,       /* CUDA launch / runtime failure              */
  PKV_E_CAPACITY = 8    /* arena too small for the requested append   */
};

#define PKV_FLAG_NONFINITE 1
#define PKV_FLAG_WIDTH 2
#define PKV_FLAG_MALFORMED 4
#define PKV_FLAG_CAPACITY 8
#define PKV_FLAG_SHAPE 16     /* score / weight row stride shorter than the token count */

#define PKV_KIND_K 0
#define PKV_KIND_V 1
#define PKV_LAYOUT_K_INTERLEAVED 0
#define PKV_LAYOUT_V_CONTIGUOUS 1

#define PKV_REPACK_NONE 0
#define PKV_REPACK_GREEDY 1
#define PKV_REPACK_V_MEDIAN 2
/* pkv_compress_tokens only: the permutation rows perm[b][nblocks_before + j]
 * of the completed block-sets are already filled in by the caller (a plan
 * computed over the heads of every shard, see pkv_repack_plan).            */
#define PKV_REPACK_EXTERNAL 3

/*
 * One layer of a batched compressed store (SPEC.md:357-362 CompressedStore,
 * one independent sub-store per layer).  `batch` sequences ×
 * `heads` KV heads = units; unit u = b*heads + h.  Blocks are `block`(=64)
 * tokens × head_dim channels, encoded per SPEC.md:330 and placed in `arena`
 * at 16-byte-aligned offsets (zero padding between blocks).
 */
typedef struct pkv_layer {
  int32_t batch;        /* sequences B                                  */
  int32_t heads;        /* KV heads per sequence H                      */
  int32_t head_dim;     /* D (32, 64, 128 or 256)                       */
  int32_t block;        /* tokens per block (64)                        */
  int32_t pack_size;    /* k in {2,4,8,16,32}                           */
  int32_t buffer;       /* staging capacity in tokens (128)             */
  int32_t max_blocks;   /* block-table capacity per unit                */
  int32_t reserved;
  uint8_t* arena;       /* append-only byte arena                       */
  int64_t arena_capacity;
  int64_t* tail;        /* [1] bytes used (16-aligned)                  */
  int64_t* blk_off;     /* [2][B*H][max_blocks] byte offset per block   */
  int32_t* blk_len;     /* [2][B*H][max_blocks] byte length per block   */
  uint8_t* perm;        /* [B][max_blocks][block] repack permutation    */
  int32_t* nblk;        /* [B] blocks per sequence                      */
  int32_t* nres;        /* [B] staged (uncompressed residue) tokens     */
  uint16_t* stage;      /* [2][B*H][buffer][D] fp16 staging ring        */
  int32_t* err;         /* [1] PKV_FLAG_* bits                          */
} pkv_layer_t;

const char* pkv_last_error(void);
int pkv_version(void);
/* Kernel family the calling thread's last fused call launched
 * (pkv_fused_k_scores / pkv_fused_v_output / pkv_attention_decode):
 * PKV_PATH_FAST = the default-format tensor-core kernels
 * (fused_{k,v}_fast_kernel), PKV_PATH_GENERIC = the scalar kernels for every
 * other format.  Lets tests assert which kernels they exercised.           */
#define PKV_PATH_NONE 0
#define PKV_PATH_FAST 1
#define PKV_PATH_GENERIC 2
#define PKV_PATH_SINGLE 3 /* pkv_attention_decode single pass (attn_fused_kernel) */
int pkv_last_path(void);

/* --- quantizer -------------------------------------- */
/* quantize_token_wise over n independent [rows, cols] fp16 tensors.
 * q: [n][rows][cols] uint16 codes; params: [n][rows][2] f32 (scale, zp). */
int pkv_quantize(const uint16_t* x, int32_t n, int32_t rows, int32_t cols, float rel,
                 uint16_t* q, float* params, int32_t* err, void* stream);
/* HalfTensor ingestion check: ORs PKV_FLAG_NONFINITE into *err
 * if any of the n fp16 values is NaN or infinite.                          */
int pkv_check_finite(const uint16_t* x, int64_t n, int32_t* err, void* stream);
/* dst = scale * src (n f32).  Either pointer may be pinned host memory (UVA:
 * the kernel reads / writes it over PCIe directly).  Plumbing of the decode
 * step's zero-copy I/O (attention_sim.GraphedAttention with host buffers): the
 * query arrives from host memory with the 1/sqrt(d) prescale applied and the
 * output leaves to host memory inside one CUDA graph.  No reference
 * counterpart (SPEC.md:520-528 takes q and returns the output; this moves them). */
int pkv_copy_scaled(const float* src, float* dst, int64_t n, float scale, void* stream);
/* dequantize: out = q*scale + zp in f32 (mul then add). */
int pkv_dequantize(const uint16_t* q, const float* params, int32_t n, int32_t rows,
                   int32_t cols, float* out, void* stream);

/* --- bitpack codec over independent blocks ------------ */
/* encode_block, pass 1: exact encoded byte length of each block.
 * q/params as produced by pkv_quantize; params may be NULL (zeros).        */
int pkv_encode_sizes(const uint16_t* q, int32_t n, int32_t rows, int32_t cols,
                     int32_t pack_size, int32_t layout, int64_t* sizes, int32_t* err,
                     void* stream);
/* encode_block, pass 2: write block i at out + offsets[i] (any alignment). */
int pkv_encode(const uint16_t* q, const float* params, int32_t n, int32_t rows, int32_t cols,
               int32_t pack_size, int32_t layout, int32_t kind, const int64_t* offsets,
               uint8_t* out, int32_t* err, void* stream);
/* decode_block: validates each header and length
 * (MalformedBlockError) and writes codes [n][rows][cols] + params f32
 * widened from the f16 wire fields.                                        */
int pkv_decode(const uint8_t* buf, const int64_t* offsets, const int64_t* lens, int32_t n,
               int32_t rows, int32_t cols, uint16_t* q, float* params, int32_t* err,
               void* stream);
/* decode_pack_at: k values of physical pack `pack_index`
 * of each block (index-range errors are raised host-side).                 */
int pkv_decode_pack_at(const uint8_t* buf, const int64_t* offsets, int32_t n, int32_t pack_index,
                       uint16_t* out, void* stream);

/* --- store: append_token / compress_batch ------------- */
/* Scratch bytes needed by pkv_compress_tokens for `nsets` block-sets.      */
int64_t pkv_compress_scratch_bytes(const pkv_layer_t* L, int32_t nsets);
/* Same for one repack strategy (PKV_REPACK_*): the default format without
 * repacking needs ~0.5 KB per block instead of the 16 KB of u16 codes.     */
int64_t pkv_compress_scratch_bytes_ex(const pkv_layer_t* L, int32_t nsets, int32_t repack);
/* append_token when it does not complete a block: stages
 * one token per sequence (k_new/v_new [B][H][D] fp16) at the device-side
 * residue count nres[b] and increments it.  Reads no host-side position, so
 * it can be captured in a CUDA graph and replayed step after step; the
 * caller runs pkv_compress_tokens for the token that completes a block.
 * nres[b] >= buffer raises PKV_FLAG_CAPACITY.                              */
int pkv_stage_token(const pkv_layer_t* L, const uint16_t* k_new, const uint16_t* v_new, void* stream);
/* Repacking across (kv-head) shards: the plan of a block-set is
 * shared by all heads of a sequence, so a rank holding some
 * heads quantizes its pending block-sets (pkv_compress_codes: codes
 * [nsets][B][2][H][block][head_dim] u16, params [...][block][2] f32 -- the
 * block-sets completed by staged + ntok tokens), all-gathers the codes of all
 * heads, computes the same plan as every other rank (pkv_repack_plan: codes
 * in the same layout with H = all heads -> perm [B][nsets][block]) and
 * compresses with PKV_REPACK_EXTERNAL.  Bytes are identical to one device
 * holding every head.                                                      */
int pkv_compress_codes(const pkv_layer_t* L, const uint16_t* k_new, const uint16_t* v_new, int32_t ntok,
                       int32_t staged, float rel_k, float rel_v, uint16_t* codes, float* params, void* stream);
/* pkv_repack_plan also backs repacker.repack_greedy / repack_v_median
 * over any 1..64 vectors (block), with a partial last
 * group when block % pack_size != 0.                        */
int pkv_repack_plan(const uint16_t* codes, int32_t nsets, int32_t batch, int32_t heads, int32_t head_dim,
                    int32_t block, int32_t pack_size, int32_t repack, uint8_t* perm, void* stream);
/* Graph-replayable flush (decode loop, default format, repack none): every
 * sequence whose staging ring holds a full block (device nres[b] >= block)
 * gets that block-set quantized, encoded and appended at the device block
 * count nblk[b] and arena tail; nblk[b] += 1, nres[b] -= block.  Sequences
 * with less staged do nothing.  Reads no host-side position, so
 * pkv_stage_token + pkv_flush_staged + pkv_attention_decode (with nblocks
 * headroom, blocks past nblk[b] are skipped) is one CUDA graph for every
 * step.  The arena must have room (PKV_FLAG_CAPACITY otherwise).  Scratch:
 * pkv_flush_scratch_bytes(L) (look-back words, ticket and epoch): zero it
 * once before the first call with it (cudaMemset); every call leaves it ready
 * for the next -- the words are tagged with a per-call epoch, so no memset
 * sits in the decode graph.  Calls sharing a scratch must be stream-ordered. */
int64_t pkv_flush_scratch_bytes(const pkv_layer_t* L);
int pkv_flush_staged(const pkv_layer_t* L, float rel_k, float rel_v, void* scratch, int64_t scratch_bytes,
                     void* stream);
/* pkv_stage_token + pkv_flush_staged in ONE launch (append_token for the
 * decode loop): each (sequence, kind, head) warp stages its
 * token at the device residue count, and a block-set the token completes is
 * compressed at once -- attention after it sees the compressed block, as the
 * reference's append_token does.  Scratch: pkv_flush_scratch_bytes, zeroed
 * once before first use (as for pkv_flush_staged).                         */
int pkv_append_flush(const pkv_layer_t* L, const uint16_t* k_new, const uint16_t* v_new, float rel_k, float rel_v,
                     void* scratch, int64_t scratch_bytes, void* stream);
/* pkv_append_flush for a ragged decode batch: only sequences with
 * active[b] != 0 (device uint8 [B]; NULL = all) append this step, so their
 * lengths diverge on the device (nblk[b], nres[b]); the fused kernels and
 * attention already follow each sequence's own counts.                     */
int pkv_append_flush_masked(const pkv_layer_t* L, const uint16_t* k_new, const uint16_t* v_new,
                            const uint8_t* active, float rel_k, float rel_v, void* scratch, int64_t scratch_bytes,
                            void* stream);
/* Appends `ntok` tokens to every sequence (lockstep batch).  k_new/v_new:
 * [B][ntok][H][D] fp16.  `staged` = tokens already staged per sequence
 * (host mirror of nres, < block); `nblocks_before` = blocks per sequence
 * before the call (host mirror of nblk).  Every full block of 64 is quantized
 * (rel_k / rel_v), repacked (`repack`, one permutation per (sequence,
 * block-set) shared by K, V and all heads), encoded (K layout
 * k_interleaved, V layout v_contiguous) and appended in arena order
 * (block-set, sequence, kind K then V, head); the remainder is staged.     */
int pkv_compress_tokens(const pkv_layer_t* L, const uint16_t* k_new, const uint16_t* v_new,
                        int32_t ntok, int32_t staged, int32_t nblocks_before, float rel_k,
                        float rel_v, int32_t repack, void* scratch, int64_t scratch_bytes,
                        void* stream);

/* --- fused decompress + GEMV --------------------------- */
/* scores[b][hq][t] = sum_c deq(K[b, hq/G][t][c]) * q[b][hq][c], t over the
 * blocks in directory (permuted-row) order then the residue; G = q_heads /
 * heads query heads share each decoded tile (GQA).  q: [B][q_heads][D] f32;
 * scores: [B][q_heads][score_stride] f32.  `nblocks` = max blocks per
 * sequence (host mirror of nblk; sizes the grid).                          */
int pkv_fused_k_scores(const pkv_layer_t* L, int32_t nblocks, const float* q, int32_t q_heads,
                       float* scores, int64_t score_stride, void* stream);
/* Scratch bytes for pkv_fused_v_output (split-L partials).                 */
int64_t pkv_fused_v_scratch_bytes(const pkv_layer_t* L, int32_t nblocks, int32_t q_heads);
/* out[b][hq][c] = sum_t w[b][hq][t] * deq(V[b, hq/G][t][c]), deterministic
 * fixed-order split-L reduction.  w: [B][q_heads][w_stride]. */
int pkv_fused_v_output(const pkv_layer_t* L, int32_t nblocks, const float* w, int32_t q_heads,
                       int64_t w_stride, float* out, void* scratch, int64_t scratch_bytes,
                       void* stream);

/* --- decode attention (SPEC.md:520-528 attention_decode) ----------------- */
/* Scratch bytes for pkv_attention_decode (0: format not fused, -1: bad args). */
int64_t pkv_attention_scratch_bytes(const pkv_layer_t* L, int32_t nblocks, int32_t q_heads);
/* out[b][hq] = softmax(scores[b][hq]) . deq(V[b, hq/G]) with
 * scores = deq(K)·q (the caller pre-scales q by 1/sqrt(d)).
 *   scores == NULL: single pass (attn_fused_kernel, §8 f1): one launch
 *     decodes K and V block by block with an online softmax per query head
 *     and merges the per-warp partials in a fixed order (deterministic); no
 *     score row ever reaches HBM.  score_stride is ignored.
 *   scores != NULL ([B][q_heads][score_stride] f32): the scores are also
 *     returned.  Three launches: fused K (also records per-slot score
 *     maxima), fused V on exp(s - M) with the row maximum M, normalising
 *     finalize.
 * q, out and scratch 16-byte aligned; calls sharing a scratch buffer must be
 * stream-ordered.  out may be pinned host memory (UVA): the last kernel
 * (finalize / merge) stores each output row to it directly.  Default format only (pack 16,
 * head_dim 128, block 64, G <= 8); else PKV_E_ARG.  Blocks past a
 * sequence's device count nblk[b] (nblocks headroom) are skipped.      */
int pkv_attention_decode(const pkv_layer_t* L, int32_t nblocks, const float* q, int32_t q_heads, float* scores,
                         int64_t score_stride, float* out, void* scratch, int64_t scratch_bytes, void* stream);

/* --- parity / debug ------------------------------------------------------ */
/* Decodes every block of one kind into codes [B*H][max_blocks][block][D]
 * (block-row order) and params [B*H][max_blocks][block][2] f32.            */
int pkv_decode_store(const pkv_layer_t* L, int32_t kind, uint16_t* codes, float* params,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PACKKV_B200_H */
