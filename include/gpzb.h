/* gpzb.h — C ABI of the B200-native GPZ compress / decompress path.
 *
 * The entry points replace the reference package's hot path
 * (/root/reference/pkg/src/gpz):
 *
 *   gpzb_compress        <- pipeline.compress            pipeline.py:73-103
 *                           (resolve_absolute_bound model.py:183-199,
 *                            _encode_block pipeline.py:38-70, compact +
 *                            write_container container.py:203-230)
 *   gpzb_range           <- model.resolve_absolute_bound model.py:183-199
 *                           + Dataset finiteness check   model.py:75-77
 *   gpzb_encode          <- the per-block map + compact  pipeline.py:78-103
 *   gpzb_parse_header    <- container.read_container     container.py:245-267
 *   gpzb_decompress      <- pipeline.decompress          pipeline.py:160-205
 *   gpzb_block_counts    <- (iter_decompressed_blocks support, pipeline.py:208-215)
 *   gpzb_pair_blocks     <- metrics.pair_blocks          metrics.py:49-81
 *   gpzb_pair_stats      <- metrics.nrmse / verify_bound metrics.py:84-152
 *
 * Conventions
 *  - Every device pointer is caller-owned (PyTorch's caching allocator in the
 *    Python host layer).  The library never allocates or frees device memory
 *    and keeps no global state; calls are re-entrant.
 *  - Work is stream-ordered on the caller's cudaStream_t (passed as void*).
 *    Functions whose name ends in _async return after enqueueing; the others
 *    synchronise the stream once at the end and read back a small result
 *    record (one D2H of < 128 bytes).
 *  - Status codes mirror gpz.errors (errors.py:4-17):
 *        0 ok, 1 DomainError, 2 WidthOverflow, 3 CorruptData,
 *        4 unsupported (valid input outside the kernels' envelope),
 *        5 invalid argument, >= 100 CUDA error.
 *    gpzb_result.block carries the first failing block (the serial
 *    first-error semantics of pipeline.py:80-83 and :183-184) or -1 for
 *    dataset/container-level errors; gpzb_reason_message() gives the text.
 */
#ifndef GPZB_H
#define GPZB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GPZB_OK 0
#define GPZB_DOMAIN_ERROR 1
#define GPZB_WIDTH_OVERFLOW 2
#define GPZB_CORRUPT_DATA 3
#define GPZB_UNSUPPORTED 4
#define GPZB_INVALID_ARGUMENT 5
#define GPZB_NEED_SIDE 6       /* gpzb_compress_result: general-encoder blocks need a side buffer
                                  of gpzb_result.side_bytes; grow it and encode again */
#define GPZB_CUDA_ERROR 100

#define GPZB_F32 0          /* model.Precision codes (model.py:29-31) */
#define GPZB_F64 1
#define GPZB_ABSOLUTE 0     /* model.EbMode codes (model.py:51-53) */
#define GPZB_RANGE_RELATIVE 1

#define GPZB_GLOBAL_HEADER_SIZE 46   /* "<4sHBBBBddIQQ", container.py:57 */
#define GPZB_MAX_BLOCK_SIZE (1u << 24) /* blocks above 1024 particles take K2b / K4b (workspace slices) */

typedef struct gpzb_result {
  int32_t status;          /* GPZB_* class of the error the reference would raise first */
  int32_t reason;          /* reason code, see gpzb_reason_message */
  int64_t block;           /* first failing block, -1 if not block-scoped */
  int32_t axis;            /* axis for per-axis reasons, else -1 */
  uint32_t nonfinite_mask; /* bit a: axis a holds non-finite values (input or output) */
  uint64_t out_len;        /* compress: container bytes; decompress: particles */
  double eb_abs;           /* compress: resolved absolute bound */
  /* raw decode diagnostics (iter_decompressed_blocks needs them separately) */
  int64_t decode_block;    /* first block failing a decode check, or -1 */
  int32_t decode_reason;
  int32_t decode_axis;
  int64_t count_block;     /* first block whose particle count breaks the boundary math, or -1 */
  uint32_t table_flags;    /* bit0 start!=0, bit1 not nondecreasing, bit2 end!=payload */
  uint32_t pad_;
  uint64_t side_bytes;     /* compress: side-buffer bytes the general-encoder blocks reserved */
  uint64_t reserved[5];
} gpzb_result;

typedef struct gpzb_header {   /* GlobalHeader, container.py:84-95 */
  uint32_t dims;
  uint32_t precision;
  uint32_t preserve_order;
  uint32_t eb_mode;
  double eb;
  double eb_abs;
  uint32_t block_size;
  uint32_t version;
  uint64_t particle_count;
  uint64_t block_count;
  uint64_t table_end;    /* 46 + 8 (block_count + 1) */
  uint64_t payload_len;  /* container length - table_end */
} gpzb_header;

/* ---- sizing ------------------------------------------------------------- */

/* Upper bound of the container length for `count` particles (the caller
 * allocates the output with it; the true length comes back in out_len). */
int gpzb_compress_bound(uint64_t count, int dims, int precision, uint32_t block_size,
                        uint32_t target_segs_per_axis, int preserve_order, uint64_t* out_bytes);

/* Device workspace needed by gpzb_compress / gpzb_range / gpzb_encode. */
int gpzb_compress_workspace(uint64_t count, int dims, int precision, uint32_t block_size,
                            uint64_t* ws_bytes);

/* Device workspace needed by gpzb_decompress for a parsed header. */
int gpzb_decompress_workspace(const gpzb_header* h, uint64_t* ws_bytes);

/* ---- compression -------------------------------------------------------- */

/* Zero the workspace's result record and look-back state (enqueued). */
int gpzb_workspace_reset_async(void* ws, uint64_t ws_bytes, uint64_t count, uint32_t block_size,
                               void* stream);

/* K1: per-block bounds + global joint range + finiteness flags (enqueued).
 * axes: `dims` device pointers to `count` coordinates each. */
int gpzb_range_async(const void* const* axes, int dims, int precision, uint64_t count,
                     uint32_t block_size, void* ws, uint64_t ws_bytes, void* stream);

/* Device address of the two int64 range words inside `ws` (order-preserving
 * encodings of -lo and +hi; all-reduce them with MAX across ranks to get the
 * global range of a sharded dataset, see DESIGN.md section multi-GPU). */
int gpzb_range_words(void* ws, uint64_t ws_bytes, int64_t** words);

/* K1.5: per-block geometry records (enqueued, after gpzb_range_async, which
 * runs in both eb modes because it also produces the per-block bounds).
 * Routes each block to the 32-bit fast encoder or the general one. */
int gpzb_encode_plan_async(const void* const* axes, int dims, int precision, uint64_t count, double eb,
                           int eb_mode, uint32_t block_size, uint32_t target_segs_per_axis,
                           int preserve_order, void* ws, uint64_t ws_bytes, void* stream);

/* The encoders and K3, enqueued after gpzb_encode_plan_async with no host
 * synchronisation in between: K2w (general blocks, into `side`), K2s / K2p /
 * K2 (32-bit fast blocks, into staging slots; every encoder is a persistent
 * kernel that reads its block list length from the device), then K3
 * (look-back scan of the payload lengths, offset table, payload moves).
 * Writes the full container (global header, offset table, payloads) into
 * `out` (capacity from gpzb_compress_bound).
 *   side / side_cap: buffer for the payloads of general-encoder blocks (may
 *   be NULL / 0).  If those blocks need more, nothing of theirs is written
 *   and gpzb_compress_result returns GPZB_NEED_SIDE with the exact size in
 *   gpzb_result.side_bytes; the caller grows the buffer and runs reset +
 *   range + plan + encode again.  Blocks take the general encoder only
 *   outside the fast path's envelope (preserve_order, > 32-bit keys,
 *   Π N > 2^16, half-bound axes).
 *   table_base / header_count / header_blocks: sharding hooks — table entries
 *   are written as table_base + local prefix, and the global header (written
 *   when write_header != 0) names header_count particles in header_blocks
 *   blocks.  Single-GPU callers pass 0, count, ceil(count/bs), 1.
 *   out == NULL: stop after the scan (K3a).  gpzb_compress_result then
 *   reports the exact container size (out_len), and gpzb_emit_async writes
 *   the container into a buffer of exactly that size — no bound-sized
 *   allocation outlives the call. */
int gpzb_encode_async(const void* const* axes, int dims, int precision, uint64_t count, double eb,
                      int eb_mode, uint32_t block_size, uint32_t target_segs_per_axis,
                      int preserve_order, void* ws, uint64_t ws_bytes, uint8_t* side,
                      uint64_t side_cap, uint8_t* out, uint64_t out_cap, uint64_t table_base,
                      uint64_t header_count, uint64_t header_blocks, int write_header, void* stream);

/* K3b after gpzb_encode_async(out == NULL) and a successful
 * gpzb_compress_result: offset table, global header (write_header != 0) and
 * payload moves into `out`, whose capacity must be the out_len that
 * gpzb_compress_result reported (the caller's claim; the payload total
 * lives on the device).  `side` is the buffer given to gpzb_encode_async.
 * Enqueued; no host synchronisation.  Replaces the concatenation step of
 * container.compact / write_container (container.py:203-230). */
int gpzb_emit_async(const void* const* axes, int dims, int precision, uint64_t count, double eb, int eb_mode,
                    uint32_t block_size, int preserve_order, void* ws, uint64_t ws_bytes, const uint8_t* side,
                    uint8_t* out, uint64_t out_cap, uint64_t table_base, uint64_t header_count,
                    uint64_t header_blocks, int write_header, void* stream);

/* Synchronise `stream` and read the result record of the last encode. */
int gpzb_compress_result(void* ws, uint64_t ws_bytes, uint64_t count, uint32_t block_size,
                         void* stream, gpzb_result* res);

/* Convenience: reset + range + plan + encode + result, one call.  A second
 * pass with a cudaMallocAsync'd side buffer runs only when general-encoder
 * blocks exist. */
int gpzb_compress(const void* const* axes, int dims, int precision, uint64_t count, double eb,
                  int eb_mode, uint32_t block_size, uint32_t target_segs_per_axis,
                  int preserve_order, void* ws, uint64_t ws_bytes, uint8_t* out,
                  uint64_t out_cap, void* stream, gpzb_result* res);

/* Diagnostics: blocks of the last compression in `ws` per encoder path,
 * counts[8]: 0 no offsets (K2, K2p), 1 composite bitmap, 2 in-group compare,
 * 3 LSD, 4 general encoder, 5 group masks or general with ranks, 6 K2s with
 * offsets, 7 K2s without offsets.  Synchronous. */
int gpzb_encode_path_counts(void* ws, uint64_t ws_bytes, uint64_t count, uint32_t block_size, int dims,
                            int precision, void* stream, uint64_t* counts);

/* ---- stage-level entry points (per-stage parity; the compress path fuses
 *      these stages into its own kernels) ---------------------------------- */

/* quantizer.block_bounds + derive_geometry (quantizer.py:51-129) for every
 * block: lohi[(blk*dims + a)*2 + {0,1}] = the block's min / max of axis a
 * (exact, as float64), Q / N = bins and segments per axis, log2m = log2 of
 * the segment size.  Any output may be NULL.  ws: gpzb_compress_workspace.
 * Synchronous; errors as in compression (non-finite input: DomainError with
 * the axis; the first failing block's WidthOverflow / DomainError). */
int gpzb_block_geometry(const void* const* axes, int dims, int precision, uint64_t count, uint32_t block_size,
                        uint32_t target_segs_per_axis, double eb_abs, double* lohi, uint64_t* Q, uint64_t* N,
                        uint8_t* log2m, void* ws, uint64_t ws_bytes, void* stream, gpzb_result* res);

/* quantizer.quantize_block (quantizer.py:223-247): the linearised
 * (seg_id, offset) of every particle, in input order, as u64 (seg and off:
 * `count` each).  lohi: NULL to use each block's own bounds, or carried
 * bounds in gpzb_block_geometry's layout (the geometry of another dataset,
 * as metrics.pair_blocks and the code fixed point use).  ws:
 * gpzb_compress_workspace.  Synchronous. */
int gpzb_quantize(const void* const* axes, int dims, int precision, uint64_t count, uint32_t block_size,
                  uint32_t target_segs_per_axis, double eb_abs, const double* lohi, uint64_t* seg, uint64_t* off,
                  void* ws, uint64_t ws_bytes, void* stream, gpzb_result* res);

/* pipeline._encode_block (pipeline.py:38-70) for every block with a given
 * absolute bound (the value compress resolves, model.py:183-199): each
 * block's serialised payload (serialize_block, container.py:98-121), back to
 * back from `payloads`, and offsets[0..nblocks] (u64 device array,
 * offsets[i] = where block i starts, offsets[nblocks] = the total) — the
 * container without its global header.  payload_cap: gpzb_compress_bound
 * minus 46 + 8 * (nblocks + 1) always suffices; when it is too small the
 * call fails with GPZB_INVALID_ARGUMENT and res->out_len = the bytes needed.
 * ws: gpzb_compress_workspace.  Synchronous; errors as compress (the first
 * failing block). */
int gpzb_encode_payloads(const void* const* axes, int dims, int precision, uint64_t count, uint32_t block_size,
                         uint32_t target_segs_per_axis, int preserve_order, double eb_abs, uint8_t* payloads,
                         uint64_t payload_cap, uint64_t* offsets, void* ws, uint64_t ws_bytes, void* stream,
                         gpzb_result* res);

/* container.compact's offsets (container.py:203-208): offsets[0] = 0,
 * offsets[i + 1] = offsets[i] + sizes[i] (u64, device arrays, nblocks + 1
 * outputs) by the K3a decoupled look-back scan.  Enqueued. */
int gpzb_scan_workspace(uint64_t nblocks, uint64_t* ws_bytes);
int gpzb_scan_sizes(const uint64_t* sizes, uint64_t nblocks, uint64_t* offsets, void* ws, uint64_t ws_bytes,
                    void* stream);

/* ---- decompression ------------------------------------------------------ */

/* Host-side validation of the 46-byte global header against the container
 * length (read_container's header checks, container.py:249-281). */
int gpzb_parse_header(const uint8_t* host_bytes, uint64_t avail, uint64_t container_len,
                      gpzb_header* h, gpzb_result* res);

/* Per-block particle counts read from the block headers (for
 * iter_decompressed_blocks' exclusive output offsets).  counts: u64[B]. */
int gpzb_block_counts_async(const uint8_t* container, uint64_t container_len,
                            const gpzb_header* h, uint64_t* counts, void* stream);

/* K4 enqueued: table validation, per-block parse + unpack + run expansion +
 * dequantize (see gpzb_decompress); read the outcome with gpzb_decompress_result. */
int gpzb_decompress_async(const uint8_t* container, uint64_t container_len, const gpzb_header* h,
                          void* const* axes_out, uint64_t out_capacity, const uint64_t* out_offsets,
                          void* ws, uint64_t ws_bytes, void* stream);

/* gpzb_decompress_async over blocks [first_block, last_block) only, so a host
 * pipeline can decode a container chunk by chunk as its bytes arrive (block
 * i reads only table entries i, i+1 and its own payload).  reset = 1 starts a
 * new decode (clears the outcome in ws); later ranges of the same container
 * pass 0 and accumulate into it, and gpzb_decompress_result then reports
 * exactly what one gpzb_decompress_async over all blocks would.  Ranges of
 * one container go on one stream, in any order. */
int gpzb_decompress_range_async(const uint8_t* container, uint64_t container_len, const gpzb_header* h,
                                void* const* axes_out, uint64_t out_capacity, const uint64_t* out_offsets,
                                void* ws, uint64_t ws_bytes, uint64_t first_block, uint64_t last_block,
                                int reset, void* stream);

/* Synchronise `stream` and classify the decode outcome in the reference's
 * precedence (table checks, first failing block, finiteness, total count). */
int gpzb_decompress_result(void* ws, uint64_t ws_bytes, const gpzb_header* h, void* stream,
                           gpzb_result* res);

/* K4: table validation, per-block parse + unpack + run expansion +
 * dequantize, written to axes_out[a][out_offsets ? out_offsets[i] : i*bs + j].
 * axes_out capacity: out_capacity particles per axis. */
int gpzb_decompress(const uint8_t* container, uint64_t container_len, const gpzb_header* h,
                    void* const* axes_out, uint64_t out_capacity, const uint64_t* out_offsets,
                    void* ws, uint64_t ws_bytes, void* stream, gpzb_result* res);

/* ---- error-bound verification (K5) --------------------------------------- */

/* Device workspace of gpzb_pair_blocks / gpzb_pair_stats for `count` pairs. */
int gpzb_pair_workspace(uint64_t count, int dims, uint64_t* ws_bytes);

/* metrics.pair_blocks (metrics.py:54-81): per block, quantize the original
 * and the reconstruction (cast to the original's precision) with the
 * original block's geometry, sort each by (seg_id, offset, index) and write
 * the positional pairing as global indices into orig_idx / rec_idx (int64,
 * `count` each).  Synchronous; errors as in compression (non-finite axis:
 * DomainError with the axis, original first; geometry: WidthOverflow with
 * the first failing block).  block_size > 1024: the sort keys live in one
 * stream-ordered scratch allocation of this call (cudaMallocAsync). */
int gpzb_pair_blocks(const void* const* orig, const void* const* rec, int dims, int precision,
                     int rec_precision, uint64_t count, double eb_abs, uint32_t block_size,
                     uint32_t target_segs_per_axis, int64_t* orig_idx, int64_t* rec_idx, void* ws,
                     uint64_t ws_bytes, void* stream, gpzb_result* res);

/* metrics.nrmse / verify_bound statistics over paired values (null index
 * arrays: identity pairing).  stats[0] = max |o - r|; per axis a:
 * stats[1 + 3a] = Σ (o - r)^2, stats[2 + 3a] = min o, stats[3 + 3a] = max o
 * (all in float64, reduced in a fixed order).  Pairs with |o - r| > eb_abs
 * are written to viol (up to viol_cap triples: axis << 56 | pair position,
 * original index, |error| bits) and counted in viol_count.  Synchronous. */
int gpzb_pair_stats(const void* const* orig, const void* const* rec, int dims, int precision,
                    int rec_precision, uint64_t count, const int64_t* orig_idx, const int64_t* rec_idx,
                    double eb_abs, uint64_t* viol, uint64_t viol_cap, void* ws, uint64_t ws_bytes,
                    void* stream, double* stats, uint64_t* viol_count);

/* ---- diagnostics -------------------------------------------------------- */

const char* gpzb_reason_message(int reason);
const char* gpzb_version(void);

/* Kernels this library has launched in the process so far (the bench
 * reports the difference over its timed region). */
uint64_t gpzb_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* GPZB_H */
