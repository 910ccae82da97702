/*
 * mergecomp.h — C ABI of the B200-native MergeComp compressed gradient-sync path.
 *
 * Drop-in boundary for the reference's codec module
 * (/root/reference/pkg/src/mergesched/compressors.py).  Every entry point is
 * extern "C", takes plain pointers and sizes (device pointers unless stated),
 * returns an int status (MC_OK = 0, negative on argument/CUDA errors) and never
 * throws.  All device work is stream-ordered on the caller's cudaStream_t
 * (passed as void*).  The library never allocates device memory (callers pass workspaces:
 * mc_encode_workspace_bytes / mc_decode_workspace_bytes) and keeps only process-wide caches
 * that do not change results: the SM count per device, per-(kernel, device) "dynamic shared
 * memory opted in" bits, a launch counter (statistics), environment tuning knobs read once,
 * and a mutex-guarded host table of randk rejection-drift statistics per (n, k) shape that
 * only sizes the speculative walk.  Data-dependent errors (non-finite gradients, corrupt indices) are
 * OR-ed into a caller-owned device word `err_flags` and surface at the
 * caller's next sync point, where the Python layer raises the reference's
 * ValueError.
 *
 * Reference interface each entry point replaces:
 *   mc_top_k_count        <- top_k_count            compressors.py:185-194
 *   mc_payload_bytes      <- payload_bytes          compressors.py:565-596
 *   mc_derive_seed        <- derive_seed            compressors.py:247-251
 *   mc_encode             <- encode (+ _compress)   compressors.py:369-417, 259-366
 *   mc_decode_mean        <- aggregate (+ decode)   compressors.py:519-532, 427-516
 *   mc_pack / mc_unpack   <- Trainer._group_slices  trainer.py:344-348 (merge stage)
 *   mc_serialize          <- serialize              compressors.py:601-620
 *   mc_deserialize        <- deserialize            compressors.py:623-645
 */
#ifndef MERGECOMP_H
#define MERGECOMP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MC_ABI_VERSION 1

/* status codes */
#define MC_OK 0
#define MC_EINVAL (-1)       /* bad argument (null pointer, n < 1, bad spec) */
#define MC_ECUDA (-2)        /* a CUDA launch or runtime call failed */
#define MC_EWORKSPACE (-3)   /* workspace smaller than mc_encode_workspace_bytes() */
#define MC_EPEER (-4)        /* the devices cannot reach each other over P2P (NVLink / PCIe) */

/* device error flags, OR-ed into *err_flags */
#define MC_ERR_NONFINITE 0x1u    /* "gradient contains non-finite values"   compressors.py:384-385 */
#define MC_ERR_INDEX_RANGE 0x2u  /* "corrupt payload: index out of range"   compressors.py:444 */
#define MC_ERR_INDEX_ORDER 0x4u  /* "corrupt payload: indices not increasing" compressors.py:445 */
#define MC_ERR_HEADER 0x8u       /* payload header does not match spec / length */
#define MC_ERR_PEER_TIMEOUT 0x10u /* mc_push_wait: a peer's payload did not arrive in time (then traps) */

/* mc_push_wait timeout when the caller passes 0: 600 s, the order of NCCL's collective timeout */
#define MC_PUSH_TIMEOUT_DEFAULT_NS 600000000000ull

/* algorithm ids == position in the reference ALGORITHMS tuple (compressors.py:29-43) */
enum {
  MC_IDENTITY = 0, MC_FP16 = 1, MC_TOPK = 2, MC_RANDK = 3, MC_DGC_LITE = 4,
  MC_THRESHOLD = 5, MC_QSGD = 6, MC_SIGNSGD = 7, MC_EFSIGNSGD = 8, MC_ONEBIT = 9,
  MC_SIGNUM = 10, MC_TERNGRAD = 11, MC_INT8 = 12, MC_NUM_ALGORITHMS = 13
};

/* Resolved CompressorSpec (compressors.py:58-107): defaults already folded in. */
typedef struct mc_spec {
  int32_t algorithm;        /* MC_* id */
  int32_t levels;           /* qsgd lattice size (>= 2) */
  int64_t bucket_size;      /* elements per scaling bucket (>= 1) */
  double sparsity;          /* dropped fraction for k-sparsifiers, [0, 1) */
  double threshold;         /* threshold codec tau (>= 0) */
  int32_t error_feedback;   /* CompressorSpec.uses_error_feedback */
  int32_t unbiased_scaling; /* randk x (n/k) */
  int32_t has_momentum;     /* CompressorSpec.momentum_coef is not None */
  float momentum;           /* float32(momentum_coef) */
} mc_spec;

/* Device payload: a 32-byte header followed by 16-byte aligned sections.
 *   idx   u32[cap]      sparsifier indices, ascending
 *   val   f32[n_val]    selected values / bucket scalers (sparse: capacity cap)
 *   bits  u8[n_bits]    sign bits (MSB-first) / packed ternary codes / fp16 / int8
 *   codes u8[n_codes]   qsgd level codes (MSB-first, width = bit_length(levels-1))
 * The canonical 22-byte-header wire form of the reference is produced by
 * mc_serialize; the aligned form is what moves through NCCL. */
typedef struct mc_payload_header {
  uint32_t algorithm;
  uint32_t flags;           /* 0x01 = randk unbiased scaling (compressors.py:55) */
  uint64_t original_len;
  uint32_t n_idx;           /* selected count (sparsifiers), else 0 */
  uint32_t n_val;
  uint32_t n_bits;          /* canonical bits length (signs + codes for qsgd) */
  uint32_t cap;             /* idx/val capacity of this buffer (sparsifiers) */
} mc_payload_header;

typedef struct mc_layout {
  int64_t n;
  int64_t cap;              /* sparse capacity (k, or n for threshold), 0 if dense */
  int64_t n_val, n_bits, n_codes;
  int64_t off_idx, off_val, off_bits, off_codes;
  int64_t bytes;            /* total device payload size, multiple of 16 */
} mc_layout;

/* Process-wide library state: a launch counter (statistics), the SM count per device
 * (cached), per-device flags of the kernel attributes already set (shared-memory opt-in),
 * and the SM reserve of mc_set_sm_reserve.  No device memory is ever allocated by the
 * library: every buffer (payloads, codec state, workspace) is the caller's. */
int mc_abi_version(void);
const char* mc_last_error(void); /* thread-local message of the last failing call */
int64_t mc_kernel_launches(void); /* kernels launched by this library since load (statistics) */
/* Size every grid for (SMs - n) so n SMs stay free for a collective running concurrently on
 * another stream (the chunked allgather pipeline's NCCL kernels); process-wide, returns the
 * previous value.  Default 0.  No reference counterpart (its allgather is a Python list). */
int mc_set_sm_reserve(int32_t n);

int64_t mc_top_k_count(double sparsity, int64_t n);
int64_t mc_payload_bytes(const mc_spec* spec, int64_t n);               /* canonical, incl. 22-B header */
int mc_payload_layout(const mc_spec* spec, int64_t n, int64_t cap, mc_layout* out); /* cap<=0: default */
int64_t mc_encode_workspace_bytes(const mc_spec* spec, int64_t n);

/* SeedSequence(entropy=(root, worker, iteration, group)).generate_state(2, u64) */
int mc_derive_seed(uint64_t root, uint64_t worker, uint64_t iteration, uint64_t group,
                   uint64_t* key_lo, uint64_t* key_hi);

/* The same keys computed on the device for a CUDA Graph that replays across iterations:
 * keys[2g], keys[2g+1] = derive_seed(root, worker, *iteration, group0 + g) for g < ngroups,
 * then *iteration += 1 (iteration: device u64; keys: device u64[2 * ngroups]).  The _dk
 * encode variants read their Philox key from such a device pair instead of (key_lo, key_hi),
 * so a captured step draws the right stream on every replay (numpy's per-(worker, iteration,
 * group) Generator, compressors.py:247-251). */
int mc_derive_keys(uint64_t root, uint64_t worker, uint64_t* iteration, uint64_t group0, int32_t ngroups,
                   uint64_t* keys, void* stream);

/* Encode one group of n fp32 gradients into `payload` (device, >= layout.bytes).
 * residual (f64[n]) must be non-null iff spec->error_feedback; momentum (f32[n])
 * iff spec->has_momentum.  Both are updated in place.  (key_lo, key_hi) is the
 * 128-bit Philox key of derive_seed() for the stochastic codecs. */
int mc_encode(const mc_spec* spec, const float* grad, int64_t n, double* residual, float* momentum,
              uint64_t key_lo, uint64_t key_hi, void* payload, void* workspace, int64_t workspace_bytes,
              uint32_t* err_flags, void* stream);

/* Single-rank sync (world size 1): encode AND out = aggregate([payload]) = 0 + decode(payload)
 * in the same pass where the codec allows it (bucketed codecs), else encode then decode.
 * `out` (f32[n]) may alias `grad` (in-place averaged gradient). */
int mc_encode_decode(const mc_spec* spec, const float* grad, int64_t n, double* residual, float* momentum,
                     uint64_t key_lo, uint64_t key_hi, void* payload, void* workspace, int64_t workspace_bytes,
                     float* out, uint32_t* err_flags, void* stream);

/* mc_encode / mc_encode_decode with the Philox key read from device memory (dkey[0..1]). */
int mc_encode_dk(const mc_spec* spec, const float* grad, int64_t n, double* residual, float* momentum,
                 const uint64_t* dkey, void* payload, void* workspace, int64_t workspace_bytes, uint32_t* err_flags,
                 void* stream);
int mc_encode_decode_dk(const mc_spec* spec, const float* grad, int64_t n, double* residual, float* momentum,
                        const uint64_t* dkey, void* payload, void* workspace, int64_t workspace_bytes, float* out,
                        uint32_t* err_flags, void* stream);

/* Chunked variant for pipelining host<->device copies with compute: encode elements
 * [begin, begin+count) of an n-element group whose buffers start at grad / residual /
 * momentum / payload / out (whole-group pointers); begin must be a multiple of the bucket
 * size and of 32, count a multiple of the bucket size unless the chunk ends the group.
 * Deterministic codecs only (identity, fp16, efsignsgd, onebit, int8); out nullable. */
int mc_encode_range(const mc_spec* spec, const float* grad, int64_t n, int64_t begin, int64_t count, double* residual,
                    float* momentum, uint64_t key_lo, uint64_t key_hi, void* payload, void* workspace,
                    int64_t workspace_bytes, float* out, uint32_t* err_flags, void* stream);

/* out[i] = (sum_{r=0..nranks-1} decode(payload_r)[i]) / f32(nranks), summed in rank
 * order in fp32 exactly as aggregate().  Payload r lives at payloads + r*stride_bytes. */
int mc_decode_mean(const mc_spec* spec, const void* payloads, int64_t stride_bytes, int32_t nranks,
                   int64_t n, float* out, uint32_t* err_flags, void* stream);
/* The same with caller-owned scratch: the sparsifiers' decode keeps a per-(rank, output tile)
 * start table of mc_decode_workspace_bytes(spec, n, nranks) bytes (0 for the dense codecs);
 * mc_decode_mean passes none and returns MC_EWORKSPACE for them.  The library never
 * allocates device memory. */
int64_t mc_decode_workspace_bytes(const mc_spec* spec, int64_t n, int32_t nranks);
int mc_decode_mean_ws(const mc_spec* spec, const void* payloads, int64_t stride_bytes, int32_t nranks, int64_t n,
                      float* out, void* workspace, int64_t workspace_bytes, uint32_t* err_flags, void* stream);

/* Merge stage: gather `count` device tensors (host array of device pointers)
 * into one contiguous buffer in list order / scatter it back. */
int mc_pack(const float* const* srcs, const int64_t* numels, int32_t count, float* fused, void* stream);
int mc_unpack(const float* fused, float* const* dsts, const int64_t* numels, int32_t count, void* stream);

/* Canonical little-endian byte form of a device payload into device `out`
 * (capacity out_cap bytes); *out_len (host) receives the byte length.  Synchronises
 * the stream for data-dependent (threshold) payloads. */
int mc_serialize(const mc_spec* spec, const void* payload, int64_t n, void* out, int64_t out_cap,
                 int64_t* out_len, void* stream);

/* Inverse of mc_serialize: canonical bytes `data` (device, `len` bytes) -> aligned device
 * payload (capacity payload_cap bytes; sparsifiers get cap = n_idx).  Validates exactly as
 * deserialize() does (short buffer, unknown algorithm id, length vs header) plus the header
 * against `spec` and its layout; *n_out (host) = original_len.  Reads the 22-byte header
 * synchronously (the section sizes depend on it). */
int mc_deserialize(const mc_spec* spec, const void* data, int64_t len, void* payload, int64_t payload_cap,
                   int64_t* n_out, void* stream);

/* Encode fused with the allgather over peer memory (NVLink P2P / symmetric memory): the
 * payload is written to `payload` (this rank's slot of its own gather buffer) and to every
 * dsts[j] (this rank's slot in rank j's gather buffer; host array of nranks device / peer-
 * mapped pointers, the entry equal to `payload` is the local one); when all of it is
 * system-visible, *flags[j] := epoch for every j (rank j's flag word for this rank).  The
 * pipe-kernel codecs (efsignsgd, onebit, int8) store into the peer slots from the encode
 * kernel itself; the others encode, then copy — threshold (data-dependent count in a
 * capacity-n slot) copies only the header and the first n_idx entries, read on the device, so
 * the variable-size exchange needs no host round trip.  mc_push_wait: the stream waits until the
 * local flags[0..nranks) all equal epoch — the gathered payloads are then complete in rank
 * order, exactly what mc_decode_mean reads (replaces the NCCL allgather of trainer.py:377-389).
 * A peer silent for timeout_ns (0 = MC_PUSH_TIMEOUT_DEFAULT_NS) sets MC_ERR_PEER_TIMEOUT and
 * traps: the stream's context faults, nothing after the wait (the decode) runs. */
int mc_encode_push(const mc_spec* spec, const float* grad, int64_t n, double* residual, float* momentum,
                   uint64_t key_lo, uint64_t key_hi, void* payload, void* const* dsts, uint32_t* const* flags,
                   int32_t nranks, uint32_t epoch, void* workspace, int64_t workspace_bytes, uint32_t* err_flags,
                   void* stream);
int mc_push_wait(const uint32_t* flags, int32_t nranks, uint32_t epoch, uint64_t timeout_ns, uint32_t* err_flags,
                 void* stream);
/* The same two calls with every per-step scalar read on the device, for a CUDA Graph of the
 * whole exchange step at N > 1: `epoch` points to the device word holding the exchange epoch
 * (the caller rewrites it before each replay), `dkey` to the Philox key (uint64[2], written by
 * mc_derive_keys at the head of the graph) — required by the codecs that draw random numbers
 * (randk, qsgd, terngrad), ignored (may be NULL) by the others. */
int mc_encode_push_dev(const mc_spec* spec, const float* grad, int64_t n, double* residual, float* momentum,
                       const uint64_t* dkey, void* payload, void* const* dsts, uint32_t* const* flags, int32_t nranks,
                       const uint32_t* epoch, void* workspace, int64_t workspace_bytes, uint32_t* err_flags,
                       void* stream);
int mc_push_wait_dev(const uint32_t* flags, int32_t nranks, const uint32_t* epoch, uint64_t timeout_ns,
                     uint32_t* err_flags, void* stream);

/* NVLink multicast (NVLS) variant of the fused push.  mc_mcast_create builds a multicast
 * object over `ndev` devices owned by this process (physical memory per device bound to it):
 * mc_mcast_ptrs gives each device's unicast view (the gather buffer its decode reads) and the
 * one multicast address.  mc_encode_push_mc encodes into `payload` (this rank's slot, unicast
 * view) with every payload word stored ONCE through `mc_slot` (the same slot's multicast
 * address: the store lands in every device's buffer), then releases `mc_flag` (multicast
 * address of this rank's flag word) := epoch on every device; mc_push_wait on a device's
 * unicast flag words then gives the gathered payloads, as with mc_encode_push.  Pipe-kernel
 * codecs (efsignsgd, onebit, int8; bucket_size % 128 == 0). */
typedef struct mc_mcast mc_mcast;
int mc_mcast_create(const int32_t* devices, int32_t ndev, int64_t bytes, mc_mcast** out);
int mc_mcast_ptrs(const mc_mcast* h, void** unicast, void** multicast, int64_t* bytes);
void mc_mcast_destroy(mc_mcast* h);
int mc_encode_push_mc(const mc_spec* spec, const float* grad, int64_t n, double* residual, float* momentum,
                      uint64_t key_lo, uint64_t key_hi, void* payload, void* mc_slot, uint32_t* mc_flag, uint32_t epoch,
                      void* workspace, int64_t workspace_bytes, uint32_t* err_flags, void* stream);

/* Peer exchange set-up (replaces nothing in the reference: its "allgather" is a Python list,
 * trainer.py:377-389).  mc_peer_enable: let kernels on `device` load/store memory of
 * `peer_device` (cudaDeviceEnablePeerAccess; a no-op when equal, MC_EPEER when the pair has
 * no P2P path).  mc_peer_probe: one kernel on the calling stream's device stores `value` to
 * every dsts[j] (peer-mapped pointers) at system scope — the store-then-readback probe that
 * proves a mapping before any encode kernel pushes through it. */
int mc_peer_enable(int32_t device, int32_t peer_device);
int mc_peer_probe(uint32_t* const* dsts, int32_t n, uint32_t value, void* stream);

/* Host-buffer sync of one rank (world size 1), enqueued natively: the trainer's step on a
 * worker's host gradient (trainer.py:360-395, one worker).  For each group: H2D of
 * host_in[0, n) into dev (device slice of the flat gradient), the fused encode + single-
 * rank aggregate in place, D2H into host_out — chunked on three streams (h2d / encode /
 * d2h) so PCIe runs full duplex; chunk c of a call waits for the previous call's read-out
 * of the same device chunk.  Chunk-wise encode for identity / fp16 / efsignsgd / onebit /
 * int8, whole-group encode between the chunked copies otherwise.  mc_pipe_finish makes
 * `s_wait` wait for the whole call; with s_wait = MC_PIPE_NO_WAIT the call keeps running
 * and the next call overlaps it (chunk-wise), until a later mc_pipe_finish with a stream
 * joins them.
 * The pipe owns only CUDA events (no device memory). */
typedef struct mc_pipe mc_pipe;
#define MC_PIPE_NO_WAIT ((void*)(intptr_t)-1)
int mc_pipe_create(mc_pipe** out);
void mc_pipe_destroy(mc_pipe* pipe);
int mc_pipe_group(mc_pipe* pipe, const mc_spec* spec, const float* host_in, float* host_out, float* dev,
                  int64_t n, int64_t chunk, double* residual, float* momentum, uint64_t key_lo, uint64_t key_hi,
                  void* payload, void* workspace, int64_t workspace_bytes, uint32_t* err_flags, void* s_h2d,
                  void* s_enc, void* s_d2h);
int mc_pipe_finish(mc_pipe* pipe, void* s_enc, void* s_d2h, void* s_wait);

#ifdef __cplusplus
}
#endif
#endif /* MERGECOMP_H */
