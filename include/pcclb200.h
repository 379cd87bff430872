/* pcclb200 -- B200-native data plane for PCCL's collectives (C ABI).
 *
 * Plain C ABI: pointers, sizes and integer codes only; no C++ exceptions
 * cross it. Every entry point returns a pcclb_status (0 = OK) unless noted.
 * Device pointers are CUDA device addresses (e.g. torch.Tensor.data_ptr());
 * `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *
 * Each entry point names the reference interface it replaces. Reference
 * paths are relative to /root/reference/pkg/src/churncomm/ (the reference is
 * pure Python/NumPy; its "FFI" for this path is the Python call seam that
 * INTEGRATION.md rebinds to this library through ctypes).
 *
 * Numerics contract: results are bit-identical to the
 * reference's NumPy arithmetic -- IEEE round-to-nearest without contraction,
 * true division, rint ties-to-even, np.maximum/np.minimum tie and NaN rules,
 * x86 NaN payload rules, no flush-to-zero.
 */
#ifndef PCCLB200_H
#define PCCLB200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PCCLB_API __attribute__((visibility("default")))
#else
#define PCCLB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------------ */
/* status codes                                                              */
/* ------------------------------------------------------------------------ */
typedef enum {
  PCCLB_OK = 0,
  PCCLB_EINVAL = 1,     /* bad argument (reference: UsageError, client.py:812-824) */
  PCCLB_ECUDA = 2,      /* CUDA runtime/driver error; see pcclb_last_cuda_error() */
  PCCLB_EABORTED = 3,   /* abort signalled; buffer restored (CollectiveAborted source="master") */
  PCCLB_ETIMEOUT = 4,   /* a peer did not arrive in time; buffer restored (source="io") */
  PCCLB_ENONFINITE = 5, /* non-finite value under quantization (collective.py:117-118);
                           buffer restored -- a documented deviation, see DESIGN.md */
  PCCLB_EIO = 6,        /* local fault injected/observed (source="io"); buffer restored */
  PCCLB_ENOMEM = 7
} pcclb_status;

/* wire.py:130-138 DType codes (only the collective dtypes) */
enum { PCCLB_F32 = 1, PCCLB_F64 = 2 };
/* Extension dtype (north_star; the reference reduces f32/f64 only, wire.py
 * DType 1/2, so parity is unpinned, oracle/bf16.py): every fold step computes
 * in f32 and rounds to bf16 (RNE). Plain ops only (quantization needs f32);
 * not sent over the reference's TCP frames. */
enum { PCCLB_BF16 = 3 };
/* wire.py:141-145 ReduceOpCode; collective.py:43-71 ReduceOp/_ACCUMULATE */
enum { PCCLB_SUM = 1, PCCLB_AVG = 2, PCCLB_MAX = 3, PCCLB_MIN = 4 };
/* Extension (north_star; absent from the reference, wire.py:141-145, so its
 * parity is unpinned): PROD folds with np.multiply in the same ring order.
 * Not sent over the reference's TCP frames (off-box peers reject it). */
enum { PCCLB_PROD = 5 };

/* Quantization formats. PCCLB_Q_U8 is the reference's (collective.py:109-135:
 * per-span min-max affine u8). The others are north_star extensions (parity
 * unpinned; oracle/quant_ext.py defines them the same way):
 *   U16:    scale = (max - min) / 65535 (1 if 0), q = u16(clip(rint((x - min) / scale)))
 *   U8_ZP / U16_ZP: min/max widened to include 0, scale = (max - min) / L (1 if 0),
 *           zp = clip(rint(-min / scale), 0, L),
 *           q = clip(rint(x / scale) + zp, 0, L), D(q) = (q - zp) * scale
 * (L = 255 / 65535; NaN -> code 0; IEEE RN, no FMA). Single-GPU seams and the
 * local ring take every format; the NVLink and TCP engines take U8 only. */
enum { PCCLB_Q_U8 = 1, PCCLB_Q_U16 = 2, PCCLB_Q_U8_ZP = 3, PCCLB_Q_U16_ZP = 4 };

/* Span range accumulator for quantization (collective.py:117-121).
 * Order-preserving u32 keys so device atomics can reduce min/max; all-zero
 * bytes is the empty range (pcclb_range_reset is a memset). kmin_inv holds
 * the bitwise complement of the minimum's key so both fields reduce with
 * atomicMax. */
typedef struct {
  uint32_t kmin_inv;
  uint32_t kmax;
  uint32_t nonfinite; /* non-zero once a NaN/Inf was seen */
  uint32_t seen;      /* non-zero once any element was seen */
} pcclb_range;

/* Per-span quantization metadata; the (min_val, scale) pair that
 * quantize_chunk returns and QuantMeta carries (collective.py:129; wire.py:844-862). */
typedef struct {
  float min_val;
  float scale;
} pcclb_qmeta;

typedef struct {
  uint64_t tx_payload_bytes; /* algorithmic bytes sent (collective.py:299,314) */
  uint64_t rx_payload_bytes; /* algorithmic bytes received (collective.py:348,368) */
  /* per-phase device time in ms when the engine was created with profiling
   * on (env PCCLB_RING_PROFILE=1); n_phases = 0 otherwise. Plain ops:
   * [copy-in, barrier0, fold, barrier1, gather(+barrier2)]; quantized ops:
   * [range, then per step (quantize, barrier, dequant-accumulate), prologue
   * + barrier, gather]. */
  uint32_t n_phases;
  float phase_ms[47];
} pcclb_stats;

PCCLB_API const char *pcclb_strerror(int status);
/* last CUDA error code seen by the library on this thread (cudaError_t) */
PCCLB_API int pcclb_last_cuda_error(void);
PCCLB_API const char *pcclb_version(void);

/* ------------------------------------------------------------------------ */
/* host-only helpers (no device work; callable without a GPU)                */
/* ------------------------------------------------------------------------ */
/* collective.py:86-101 compute_chunk_boundaries: out[2*r] = lo, out[2*r+1] = hi */
PCCLB_API int pcclb_chunk_bounds(uint64_t n_elements, uint32_t world_size, uint64_t *out_lo_hi);

/* ------------------------------------------------------------------------ */
/* kernel seams (single GPU)                                                 */
/* ------------------------------------------------------------------------ */
/* collective.py:66-71,407,416: acc <- acc (+) in  (np.add / np.maximum / np.minimum) */
PCCLB_API int pcclb_accumulate(void *acc, const void *in, uint64_t n, int dtype, int op, void *stream);

/* collective.py:479-482 finalize_reduction: AVG -> buf /= dtype(world); else no-op */
PCCLB_API int pcclb_finalize(void *buf, uint64_t n, int dtype, int op, uint32_t world, void *stream);

/* quantize_chunk range part (collective.py:117-121) */
PCCLB_API int pcclb_range_reset(pcclb_range *d_range, uint32_t count, void *stream);
PCCLB_API int pcclb_range_f32(const float *x, uint64_t n, pcclb_range *d_range, void *stream);

/* quantize_chunk map part (collective.py:119-129): codes = Q(x) using the
 * range in d_range; writes (min_val, scale) to d_meta (empty span: (0, 1)).
 * adopt_out (nullable): adopt_out = D(codes) / avg_div (avg_div = 1 for none) --
 * the owner adoption of collective.py:538-551 fused with finalize. */
PCCLB_API int pcclb_quantize_u8(const float *x, uint64_t n, const pcclb_range *d_range, uint8_t *codes,
                      pcclb_qmeta *d_meta, float *adopt_out, uint32_t avg_div, void *stream);

/* collective.py:132-135 dequantize_into (+ optional fused AVG finalize) */
PCCLB_API int pcclb_dequantize_u8(float *out, const uint8_t *codes, uint64_t n, const pcclb_qmeta *d_meta,
                        uint32_t avg_div, void *stream);

/* collective.py:399-409 quantized consume: acc <- acc (+) D(codes); if d_next_range is
 * non-null the range of the new acc is accumulated there (fused K2). */
PCCLB_API int pcclb_dequant_accumulate_u8(float *acc, const uint8_t *codes, uint64_t n,
                                const pcclb_qmeta *d_meta, int op, pcclb_range *d_next_range,
                                void *stream);
/* The three seams for any quantization format (PCCLB_Q_*; codes are u8 or
 * u16 per format; for the _ZP formats d_meta->min_val holds the zero point).
 * PCCLB_Q_U8 forwards to the _u8 functions above. */
PCCLB_API int pcclb_quantize_ex(const float *x, uint64_t n, const pcclb_range *d_range, void *codes,
                                pcclb_qmeta *d_meta, float *adopt_out, uint32_t avg_div, int qformat, void *stream);
PCCLB_API int pcclb_dequantize_ex(float *out, const void *codes, uint64_t n, const pcclb_qmeta *d_meta,
                                  uint32_t avg_div, int qformat, void *stream);
PCCLB_API int pcclb_dequant_accumulate_ex(float *acc, const void *codes, uint64_t n, const pcclb_qmeta *d_meta,
                                          int op, pcclb_range *d_next_range, int qformat, void *stream);

/* Outer-optimizer steps of the DiLoCo loops around the all-reduce, with the
 * reference's rounding sequence (algos.py:79-105, :236-239):
 * delta = global - local; PlainSGD params -= lr * grad;
 * NesterovOuter v = v*mu; v = v + delta; params -= lr * (delta + mu*v). */
PCCLB_API int pcclb_pseudo_gradient_f32(float *delta, const float *global, const float *local,
                                        uint64_t n, void *stream);
PCCLB_API int pcclb_outer_sgd_f32(float *params, const float *grad, uint64_t n, float lr,
                                  void *stream);
PCCLB_API int pcclb_outer_nesterov_f32(float *params, const float *delta, float *velocity,
                                       uint64_t n, float lr, float momentum, void *stream);

/* sharedstate.py:87-105 simplehash over one device buffer; result to d_out[0] */
PCCLB_API int pcclb_simplehash(const void *d_data, uint64_t nbytes, uint64_t *d_out, void *stream);

/* simplehash of `count` device buffers in one persistent launch (largest-first
 * dynamic scheduling); sharedstate.py:171-178 content_hash / digest_entries.
 * h_ptrs/h_nbytes are host arrays; d_out is a device array of `count` u64. */
PCCLB_API int pcclb_simplehash_multi(const void *const *h_ptrs, const uint64_t *h_nbytes, uint32_t count,
                           uint64_t *d_out, void *stream);

/* Resumable simplehash for streaming an entry through device memory in pieces
 * (e2e path: host->device copy of segment i+1 overlaps hashing of segment i).
 * d_state holds 256 u64 lane values; every segment except the last must be a
 * multiple of 1024 bytes. pcclb_simplehash_final folds lanes and XORs total_nbytes. */
PCCLB_API int pcclb_simplehash_init(uint64_t *d_state, void *stream);
PCCLB_API int pcclb_simplehash_update(uint64_t *d_state, const void *d_data, uint64_t nbytes, void *stream);
PCCLB_API int pcclb_simplehash_final(const uint64_t *d_state, uint64_t total_nbytes, uint64_t *d_out,
                           void *stream);

/* CRC-32 digests (extension: the north_star's "simplehash/CRC32"; absent from
 * the reference). zlib.crc32 of each device buffer -- reflected polynomial
 * 0xEDB88320, init and final xor 0xFFFFFFFF -- written to d_out[i] (uint32).
 * One launch for all entries (256 KiB segments per CTA, combined with
 * GF(2) shifts). Parity is pinned by zlib itself. */
PCCLB_API int pcclb_crc32_multi(const void *const *h_ptrs, const uint64_t *h_nbytes, uint32_t count,
                                uint32_t *d_out, void *stream);
PCCLB_API int pcclb_crc32(const void *d_data, uint64_t nbytes, uint32_t *d_out, void *stream);

/* ------------------------------------------------------------------------ */
/* local ring: W logical peers whose buffers live on ONE GPU                 */
/* (the reference's in-process RingSession, tests/ring_harness.py:24-105)    */
/* ------------------------------------------------------------------------ */
/* Runs run_all_reduce (collective.py:489-567) for W ring positions at once.
 * h_bufs: host array of W device pointers, ring-position order, each n elements.
 * d_scratch: device scratch of at least pcclb_local_scratch_bytes(w) bytes.
 * Returns PCCLB_ENONFINITE (buffers untouched if d_backup given, see below)
 * when a quantized span is non-finite. d_backup (nullable): W*n elements
 * used to restore the buffers on failure (collective.py:501-504, :568-574). */
PCCLB_API uint64_t pcclb_local_scratch_bytes(uint32_t world);
PCCLB_API int pcclb_local_allreduce(void *const *h_bufs, uint32_t world, uint64_t n, int dtype, int op,
                          int quantize, void *d_scratch, void *d_backup, void *stream);
/* Same with a quantization format (0 = none, PCCLB_Q_*). */
PCCLB_API int pcclb_local_allreduce_ex(void *const *h_bufs, uint32_t w, uint64_t n, int dtype, int op,
                                       int qformat, void *d_scratch, void *d_backup, void *stream);

/* ------------------------------------------------------------------------ */
/* intra-box ring over NVLink: one process per GPU                           */
/* ------------------------------------------------------------------------ */
typedef struct pcclb_ring pcclb_ring;

/* Create the engine for ring position `rank` of `world` on CUDA device
 * `device`. Allocates an IPC-exportable workspace of `capacity_bytes`. */
PCCLB_API int pcclb_ring_create(int device, uint32_t rank, uint32_t world, uint64_t capacity_bytes,
                      pcclb_ring **out);
/* 64-byte cudaIpcMemHandle of this rank's workspace (exchange out of band). */
PCCLB_API int pcclb_ring_export(pcclb_ring *r, void *handle64_out);
/* Map peer `peer`'s workspace (handle from its pcclb_ring_export). */
PCCLB_API int pcclb_ring_import(pcclb_ring *r, uint32_t peer, const void *handle64);
/* Host-mapped abort word the control plane may set (reference: the tag box
 * abort_event set on ABORT_NOTIFY, client.py:196-204). Returns host pointer.
 * Attempt-scoped: storing A aborts every attempt <= A at its next barrier,
 * vote or fused-step poll; later attempts are unaffected (no reset needed). */
PCCLB_API volatile uint64_t *pcclb_ring_abort_word(pcclb_ring *r);
/* Number of engines that may run ops concurrently on this GPU (the
 * communicator's pool of slots, client.py:482-486; default 2). The fused
 * quantized steps spin on peer-ready flags with persistent CTAs, so each engine
 * takes at most its share of the SM's CTA slots; with more engines than slots
 * the engine falls back to one barrier per ring step. */
PCCLB_API int pcclb_ring_set_slots(pcclb_ring *r, uint32_t slots);
/* Plain ops of at most `bytes` run as one fused kernel (copy-in, arrival,
 * local fold of every chunk in its ring order, completion vote): the
 * latency-bound end of the config-2 sweep. Default 64 MiB at W = 2, else 32 MiB / W
 * (PCCLB_SMALL_MAX overrides); 0 disables. Every rank of a ring must use the same value (the
 * path is part of the parameter check at the arrival). */
PCCLB_API int pcclb_ring_set_small_max(pcclb_ring *r, uint64_t bytes);
/* Workspace bytes an n-element op needs at this world size (host-only, no
 * GPU needed): the capacity_bytes to pass to pcclb_ring_create. 0 if invalid. */
PCCLB_API uint64_t pcclb_ring_workspace_bytes(uint64_t n, uint32_t world, int dtype, int quantize);
/* Element capacity for a dtype/quantize combination with this workspace. */
PCCLB_API uint64_t pcclb_ring_capacity(pcclb_ring *r, int dtype, int quantize);

/* Caller-buffer registration (collective: every rank registers the same
 * logical buffers in the same slot order). pcclb_ipc_handle gives the CUDA IPC
 * handle of the allocation holding d_ptr and d_ptr's offset in it; after an
 * out-of-band exchange, pcclb_ring_register maps every peer's buffer
 * (handles: world x 64 bytes and offsets: world entries, ring-position order).
 * All-reduces on a registered buffer read it in place over NVLink instead of
 * staging a copy (the backup copy then overlaps the fold). */
PCCLB_API int pcclb_ipc_handle(const void *d_ptr, void *handle64_out, uint64_t *offset_out);
PCCLB_API int pcclb_ring_register(pcclb_ring *r, uint32_t slot, const void *local_ptr,
                                  uint64_t nbytes, const void *handles, const uint64_t *offsets);
PCCLB_API int pcclb_ring_deregister(pcclb_ring *r, uint32_t slot);

/* run_all_reduce (collective.py:489-576) on this rank's buffer. `attempt` must
 * be identical on all ranks and strictly increasing per engine (the reference's
 * (tag, seq_nr) attempt identity, collective.py:343-356). `fault_at` >= 0
 * injects a local fault at that synchronisation point (reference fault_hook,
 * collective.py:268-272); -1 disables. Blocks until the op resolves. On any
 * failure the buffer is restored byte-exactly before returning. */
PCCLB_API int pcclb_ring_allreduce(pcclb_ring *r, void *d_buf, uint64_t n, int dtype, int op,
                         int quantize, uint64_t attempt, int fault_at, double timeout_s,
                         pcclb_stats *out_stats, void *stream);
/* Peer memory for shared-state resync (client.py:743-798 fetches an entry
 * from its donor): map a peer allocation by its IPC handle (refcounted per
 * process), and copy device/peer bytes on a stream (NVLink for peer memory). */
PCCLB_API int pcclb_ipc_open(const void *handle64, void **ptr_out);
PCCLB_API int pcclb_ipc_close(void *ptr);
PCCLB_API int pcclb_copy(void *dst, const void *src, uint64_t bytes, void *stream);

/* Asynchronous form (all_reduce_async / await_async_reduce, client.py:802-843):
 * enqueue returns a ticket once every kernel of the op is on `stream`; wait
 * blocks until it resolves and returns the same statuses as
 * pcclb_ring_allreduce (which is enqueue + wait). Up to 64 ops may be
 * outstanding; ops on one stream run in order. */
PCCLB_API int pcclb_ring_enqueue(pcclb_ring *r, void *d_buf, uint64_t n, int dtype, int op,
                                 int quantize, uint64_t attempt, int fault_at, double timeout_s,
                                 void *stream, uint32_t *ticket_out);
PCCLB_API int pcclb_ring_wait(pcclb_ring *r, uint32_t ticket, pcclb_stats *out_stats);
/* Restore the last op's input (completion-vote veto, client.py:973-983).
 * Valid until the next pcclb_ring_allreduce on this engine. */
PCCLB_API int pcclb_ring_restore(pcclb_ring *r, void *d_buf, uint64_t n, int dtype, void *stream);
PCCLB_API void pcclb_ring_destroy(pcclb_ring *r);

#ifdef __cplusplus
}
#endif
#endif /* PCCLB200_H */
