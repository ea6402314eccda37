/*
 * zipccl_b200.h — C-ABI of libzipccl_b200.so, the B200 (sm_100a) hot path of
 * ZipCCL (arxiv 2604.27844): lossless BF16 exponent coding and the pieces of
 * the compressed all-gather / all-to-all that run on the device.
 *
 * The reference (/root/reference/pkg/src/zipcoll, pure Python + NumPy) has no
 * native boundary; its plugin surface is the Python package API.  Each entry
 * point below names the reference function it replaces.  A Python binding
 * (ctypes) lives in paper_2604_27844_b200/_lib.py; INTEGRATION.md shows how a
 * maintainer wires the reference package onto it.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless stated; host arrays are marked
 *     "host".  BF16 data are 16-bit words (bit patterns, never values).
 *   - Work is enqueued on `stream` (a cudaStream_t passed as void*); no entry
 *     point synchronises with the host.
 *   - Return value: 0 ok; -1 invalid argument; -2 workspace too small;
 *     -3 frame would exceed the u32 offset range (reference
 *     UnrepresentableError, container.py:76-78); >0 a cudaError_t.
 *   - Frames are byte-identical to
 *     container.serialize(codec.compress(x, book, 1 << gs_log2)).
 */
#ifndef ZIPCCL_B200_H
#define ZIPCCL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI version (2). */
int zc_abi_version(void);
/* Kernel timing hooks (measurement only).  zc_profile_enable(1) resets and
 * starts recording CUDA events on the launching stream around every pass-1
 * encoder launch (tag 0; zc_encode / zc_encode_measured) and every decoder
 * launch (tag 1; zc_decode); zc_profile_enable(0) stops.  Never enable while
 * a stream is being captured into a CUDA graph.  zc_profile_read waits for
 * the recorded events and writes up to `cap` launch durations (ms) of `tag`
 * into ms; returns how many (or a negative status). */
int zc_profile_enable(int on);
int zc_profile_read(int tag, float* ms, int cap);

/* Elements per CTA tile of the encode/decode/stats kernels (4096). */
int zc_tile_elements(void);
/* Segments accepted per batched call (64). */
int zc_max_segments(void);
/* Human-readable text for a status code. */
const char* zc_status_string(int status);

/* Replaces codec.static_size_bytes (codec.py:381-395): bytes of the static
 * part [header .. group_index] of a frame of n elements; -1 if invalid. */
int64_t zc_static_bytes(int64_t n, int gs_log2);

/* Upper bound of a frame (every element escaping): static + pad128(n)
 * (codec.compressed_size_bytes, codec.py:398-401, with zero_count = n). */
int64_t zc_max_frame_bytes(int64_t n, int gs_log2);

/* Device scratch needed by any call below over `total_elems` elements in
 * `nseg` segments. */
int64_t zc_workspace_bytes(int64_t total_elems, int nseg);

/* Replaces codec.codebook_for(data, sigma=None) (codec.py:164-185) with
 * bf16.measure_sigma (bf16.py:88-103), over the concatenation of the segments
 * x[seg_off[i] : seg_off[i]+seg_n[i]] (host arrays; empty segments skipped) —
 * the all-to-all scope of collectives._prepare_frames (collectives.py:230-242).
 * Writes book_dev[0..6] = entries, book_dev[7] = 0 and
 * result_dev[0] = sigma (NaN if no finite element), result_dev[1] = finite
 * count, result_dev[2] = 1 (analytic) / 2 (modal fallback) / 3 (analytic,
 * certified).  Without ZC_SIGMA_EXACT in `flags` a packed-fp32 pass with a
 * rigorous error bound decides the codebook whenever the whole sigma
 * interval maps to one codebook (path 3, result_dev[0] then within ~2e-6
 * relative of the f64 statistic); otherwise, and always with
 * ZC_SIGMA_EXACT, the f64 pass runs (paths 1/2).  The codebook is the
 * reference's either way. */
#define ZC_SIGMA_EXACT 1
int zc_codebook_measured(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n,
                         int nseg, void* ws, int64_t ws_bytes, uint8_t* book_dev,
                         double* result_dev, int flags, void* stream);

/* Replaces the modal fallback of codec.codebook_for for an explicit sigma that
 * is 0, negative or non-finite (codec.py:179-185): window around the first
 * argmax of the 256-bin exponent histogram. */
int zc_codebook_modal(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n, int nseg,
                      void* ws, int64_t ws_bytes, uint8_t* book_dev, void* stream);

/* Replaces container.serialize(codec.compress(chunk, book, 1 << gs_log2))
 * (codec.py:264-305, container.py:65-95) — and, with nseg > 1, the per-peer
 * framing loop of collectives._prepare_frames (collectives.py:241-242).
 * Segment i (host arrays seg_off/seg_n/frame_off, seg_n[i] >= 1) is encoded
 * into frames + frame_off[i] (128-byte aligned, capacity
 * zc_max_frame_bytes(seg_n[i])); frame_len_dev[i] receives its length. */
int zc_encode(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n,
              const int64_t* frame_off, int nseg, const uint8_t* book_dev, int gs_log2,
              uint8_t* frames, void* ws, int64_t ws_bytes, uint64_t* frame_len_dev,
              void* stream);

/* Replaces container.serialize(codec.compress(x, codec.codebook_for(x)))
 * (codec.py:164-185 + :264-305) — and for nseg > 1 the whole of
 * collectives._prepare_frames (collectives.py:230-242): ONE codebook measured
 * over the concatenation of the segments, one frame per segment.  flags bit 0
 * (ZC_ENCODE_SPECULATIVE, what the Python layer passes) selects the
 * speculative path for inputs of >= 1024 tiles: a codebook guessed from a
 * uniform 1/128 sample, the encoder run with it while it accumulates the
 * certified packed-fp32 statistic of all of x, the exact f64 pass only if the
 * certificate fails and a re-encode only if the exact codebook differs from
 * the guess -- identical output, one pass over x fewer (measured 176 vs
 * 237 us at 218M words when introduced; 166 us now).  book_dev / result_dev receive the exact codebook
 * and (sigma, finite count, path) like zc_codebook_measured. */
#define ZC_ENCODE_SPECULATIVE 1
int zc_encode_measured(const uint16_t* x, const int64_t* seg_off, const int64_t* seg_n,
                       const int64_t* frame_off, int nseg, int gs_log2, uint8_t* frames, void* ws,
                       int64_t ws_bytes, uint64_t* frame_len_dev, uint8_t* book_dev,
                       double* result_dev, int flags, void* stream);

/* Replaces codec.decompress(container.parse(frame)) (container.py:113-180,
 * codec.py:210-327) per segment, i.e. collectives._parse_peer_frame
 * (collectives.py:185-200).  stat[i] = frame start (16-byte aligned, may be a
 * peer-mapped address), dyn[i] = zero-exponent section (NULL: in place after
 * the static part, the design-2 split otherwise), dyn_len[i] = bytes of that
 * section (-1 unknown; host array may be NULL), n[i] = expected element count,
 * out_off[i] = element offset of the output.  err_dev[i] = 0x7F7F7F7F when the
 * frame is valid, else the smallest failing check in reference order
 * (see engine.ERR_FIELDS).  write_out = 0 validates only (reference
 * CompressedChunk.validate, codec.py:252-255). */
int zc_decode(const uint8_t* const* stat, const uint8_t* const* dyn, const int64_t* dyn_len,
              const int64_t* n, const int64_t* out_off, int nseg, uint16_t* out,
              int32_t* err_dev, void* ws, int64_t ws_bytes, int write_out, void* stream);

/* Replaces codec.decompress_group (codec.py:330-348), generalised to a
 * range: the words of groups [g0, g1) of a frame of n elements with group
 * size 1 << gs_log2 are written to out[0 ..), reading only those groups'
 * sign-mantissa / plane bytes and their escapes (from group_index[g0]).
 * The frame's structure must have been validated (zc_decode with
 * write_out = 0, as the reference validates first); escape positions are
 * clamped, so a corrupt frame cannot cause out-of-bounds reads.  frame is
 * 8-byte aligned. */
int zc_decode_groups(const uint8_t* frame, int64_t n, int gs_log2, int64_t g0, int64_t g1,
                     uint16_t* out, void* stream);

/* ---- peer memory for the compressed collectives over NVLink -------------
 * Replace the transport seam (transport.Communicator send/recv,
 * transport.py:559-623) for the pull-decode all-gather / all-to-all:
 * frames stay in each rank's HBM and peers decode them in place. */

/* Size of an IPC handle blob (64). */
int zc_ipc_handle_bytes(void);
/* Export the allocation containing dev_ptr into handle_out (host, 64 B). */
int zc_ipc_get_handle(void* dev_ptr, void* handle_out);
/* Map a peer's exported allocation; *dev_ptr_out = its base in this process. */
int zc_ipc_open_handle(const void* handle, void** dev_ptr_out);
/* Unmap a pointer returned by zc_ipc_open_handle. */
int zc_ipc_close_handle(void* dev_ptr);
/* cudaMalloc'd, zero-filled buffer outside the framework's caching allocator
 * (so an IPC handle maps exactly this allocation). */
int zc_alloc(int64_t bytes, void** dev_ptr_out);
int zc_free(void* dev_ptr);
/* Device-side signal: write `epoch` into slot `my_rank` of every peer's flag
 * array (peer_flags: host array of world device pointers). */
int zc_signal_peers(void* const* peer_flags, int world, int my_rank, uint64_t epoch, void* stream);
/* Device-side wait until flags[p] >= epoch for every p != my_rank (or the
 * clock-based timeout in ns expires: err_dev = 20). */
int zc_wait_signals(const void* flags, int world, int my_rank, uint64_t epoch,
                    int64_t timeout_ns, int32_t* err_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ZIPCCL_B200_H */
