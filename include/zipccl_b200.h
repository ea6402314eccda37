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
 * uniform 1/512 sample, the encoder run with it while it accumulates the
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
 * (see engine.ERR_FIELDS).  write_out bit 0 clear validates only (reference
 * CompressedChunk.validate, codec.py:252-255); bit 1: frames may use groups
 * larger than 4096 elements; bit 3 (ZC_DECODE_GROUPS512): the caller knows
 * every frame uses 512-element groups, so frames of at most 512 Ki elements
 * are decoded by one cluster launch (a frame with another group size then
 * fails with code 22). */
#define ZC_DECODE_GROUPS512 8
int zc_decode(const uint8_t* const* stat, const uint8_t* const* dyn, const int64_t* dyn_len,
              const int64_t* n, const int64_t* out_off, int nseg, uint16_t* out,
              int32_t* err_dev, void* ws, int64_t ws_bytes, int write_out, void* stream);

/* Decode behind arrival: the per-peer decode of the reference's receive
 * loop (collectives.py:216-227) as ONE launch over frames that are still
 * arriving.  Frame s (its static part at stat[s], 16-B aligned, the dynamic
 * section in place) is decoded once *ready[s] >= epoch (acquire load at
 * system scope; the writer publishes after its frame with a release store or
 * a completed copy), in whatever order the flags appear: work on the frames
 * already complete proceeds while later ones are in flight.  Frames of n[s]
 * elements with groups of <= 4096 elements; words to out + out_off[s].
 * err_dev[s] as zc_decode; 20 if the flag did not arrive within timeout_ns
 * (0: wait forever).  ws >= zc_workspace_bytes(sum n, nseg). */
int zc_decode_when_ready(const uint8_t* const* stat, const int64_t* n, const int64_t* out_off,
                         const uint64_t* const* ready, int nseg, uint64_t epoch,
                         int64_t timeout_ns, uint16_t* out, int32_t* err_dev, void* ws,
                         int64_t ws_bytes, void* stream);

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

/* ---- ratio estimate (adaptive switch) ----------------------------------------
 * Estimated frame bytes / raw bytes of compressing x[0, n) under the codebook
 * codebook_for would pick (sampled; at least 2^22 words, at most 1/64 of the
 * bytes): out_dev[0] = e, [1] = sample sigma, [2] = sample escape fraction.
 * Feeds the message-adaptive switch (switcher.select with the message's e;
 * reference switcher.py:83-95 uses one profiled e).  ws >= 4096 bytes. */
int zc_estimate_ratio(const uint16_t* x, int64_t n, void* ws, double* out_dev, void* stream);

/* ---- fused decode + fp32 reduction (reduce-scatter) ---------------------------
 * Replaces collectives._reduce_chunks over decoded peer chunks
 * (collectives.py:137-144, :328-341; narrowing bf16.from_float32, bf16.py:53-66):
 * out = sum over sources in list order, float32 adds with numpy's x86 NaN
 * semantics, then RNE with the quiet bit forced (out_f32: the float32 sums).
 * src_dev: device array of W records of zc_red_src_bytes() bytes each,
 *   { const uint8_t* stat; const uint8_t* dyn; int64_t dyn_len;
 *     const uint64_t* ready; int32_t raw; int32_t pad; }
 * (raw != 0: stat points at n raw words; else a frame of n elements with
 * 512-element groups, dyn = split zero-exponent section or NULL).
 * err_dev[W] = 0x7F7F7F7F per valid source, else the failing check. */
int zc_red_src_bytes(void);
int64_t zc_reduce_scratch_bytes(int W);
int zc_reduce_frames(const void* src_dev, int W, int64_t n, void* out, int out_f32,
                     void* hdr_scratch, int32_t* err_dev, void* stream);

/* ---- native compressed collectives (csrc/zc_coll.cu) ---------------------------
 * Replace the reference's collectives over its transport seam
 * (collectives.zip_all_gather :203-227, zip_all_to_all_d1/_d2 :245-325,
 * zip_reduce_scatter :328-341, reference_* :97-170; Communicator
 * transport.py:576-623) with C++ over NCCL and CUDA peer memory.
 *
 * A communicator is one rank of a group: zc_comm_init bootstraps it from an
 * NCCL unique id (rank 0 calls zc_nccl_get_id and distributes the bytes, as
 * with ncclCommInitRank); zc_comm_init_local creates all ranks of an
 * in-process group (one host thread drives each rank afterwards).  Every
 * rank owns a symmetric buffer (2 frame slots of slot_bytes + flags) that
 * its peers map (CUDA IPC / direct pointers); when all mappings succeed the
 * peer-memory plane is available.
 *
 * Collective calls are stream-ordered on `stream` and do not synchronise
 * with the host on the peer-memory plane; the message plane reads the frame
 * sizes back (the reference's size phase).  err_dev[world] (int32, device)
 * receives 0x7F7F7F7F per peer whose frame decoded, else the failing check
 * (engine.ERR_FIELDS; 19 = element count differs, 20 = peer never ready).
 * book_dev: uint8[8] codebook on the device, or NULL for codebook_for
 * semantics (sigma measured over the chunks sent).
 * Status: 0 ok, -1 bad argument, -3 frame too large (UnrepresentableError),
 * -4 sizes/counts disagree (ProtocolError), -5 peer-memory region too small
 * for this all-to-all (grow with zc_comm_reserve), -6 transport failure,
 * -7 a peer's frame is unusable (CollectiveError; zc_comm_last_error gives
 * the message and the peer), > 0 a cudaError_t. */
typedef struct zc_comm zc_comm;

#define ZC_PLANE_P2P 1      /* peer-memory plane (default when available) */
#define ZC_PLANE_MSG 2      /* message plane: reference protocols over NCCL */
#define ZC_A2A_D1 4         /* all-to-all design 1 (metadata + frames), message plane */
#define ZC_CHECK_COUNTS 8   /* agree element counts first (NCCL cannot detect mismatches) */
#define ZC_PIPELINE 16      /* message-plane all-gather: ring steps, per-peer decode on a side stream */
#define ZC_COMM_NO_P2P 1    /* zc_comm_init flags: never use the peer-memory plane */

int zc_nccl_id_bytes(void);
int zc_nccl_get_id(void* id_out);
/* rank of world over NCCL; device = the current CUDA device.  slot_bytes:
 * peer-memory slot capacity (<= 0: 256 MiB; all-gather slots grow
 * collectively, all-to-all regions are slot_bytes / world per peer). */
int zc_comm_init(zc_comm** comm, const void* nccl_id, int rank, int world, int64_t slot_bytes,
                 int flags);
/* world in-process ranks; devices[i] is rank i's CUDA device (NULL: current). */
int zc_comm_init_local(zc_comm** comms, int world, const int* devices, int64_t slot_bytes,
                       int flags);
int zc_comm_destroy(zc_comm* comm);
/* releases in-process ranks blocked in a rendezvous after a peer failed */
int zc_comm_abort(zc_comm* comm);
/* info[5] = rank, world, peer-memory plane available, a peer shares this
 * device, NCCL-backed */
int zc_comm_info(zc_comm* comm, int* info);
const char* zc_comm_last_error(zc_comm* comm, int* peer);
/* TrafficStats (transport.py:559-573): bytes / messages this rank sent
 * (synchronises the device to read the peer-memory plane's counters) */
int zc_comm_stats(zc_comm* comm, uint64_t* bytes_sent, uint64_t* messages);
/* collectively grow the peer-memory slots (every rank, same value) */
int zc_comm_reserve(zc_comm* comm, int64_t slot_bytes, void* stream);

/* zip_all_gather: out[p*n ..] = rank p's x (n >= 1 on every rank) */
int zc_allgather(zc_comm* comm, const uint16_t* x, int64_t n, uint16_t* out,
                 const uint8_t* book_dev, int32_t* err_dev, int flags, void* stream);
/* reference_all_gather's data movement: ncclAllGather of the words */
int zc_allgather_raw(zc_comm* comm, const uint16_t* x, int64_t n, uint16_t* out, void* stream);
/* zip_all_to_all: x = send chunks back to back (send_counts[world] words,
 * host array), out = receive chunks back to back (recv_counts[world];
 * recv_counts[rank] must equal send_counts[rank]).  Peer-memory plane, or
 * the message plane with design 2 (default) / design 1 (ZC_A2A_D1). */
int zc_alltoall(zc_comm* comm, const uint16_t* x, const int64_t* send_counts,
                const int64_t* recv_counts, uint16_t* out, const uint8_t* book_dev,
                int32_t* err_dev, int flags, void* stream);
int zc_alltoall_raw(zc_comm* comm, const uint16_t* x, const int64_t* send_counts,
                    const int64_t* recv_counts, uint16_t* out, int flags, void* stream);
/* zip_reduce_scatter: x = world shards of `shard` words; out = this rank's
 * shard reduced over ranks in ascending order (bf16 words, or float32 with
 * out_f32) by the fused decode + reduce kernel */
int zc_reduce_scatter(zc_comm* comm, const uint16_t* x, int64_t shard, void* out, int out_f32,
                      const uint8_t* book_dev, int32_t* err_dev, int flags, void* stream);
int zc_reduce_scatter_raw(zc_comm* comm, const uint16_t* x, int64_t shard, void* out,
                          int out_f32, int32_t* err_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ZIPCCL_B200_H */
