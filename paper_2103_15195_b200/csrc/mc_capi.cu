// mc_capi.cu — the extern "C" boundary (include/mergecomp.h): argument validation,
// payload layout, SeedSequence key derivation and dispatch to the codec kernels.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>

#include "mc_internal.cuh"

namespace mc {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static std::atomic<int> g_sm_reserve{0};  // SMs left to a concurrent collective (mc_set_sm_reserve)

// SMs the library sizes its grids for: the device's count less the reserve
int sm_count() {
  static std::atomic<int> cached[64];  // per device (zero = not read yet)
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& c = cached[dev & 63];
  int v = c.load(std::memory_order_relaxed);
  if (!v) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    c.store(v, std::memory_order_relaxed);
  }
  const int r = g_sm_reserve.load(std::memory_order_relaxed);
  return v - r >= 1 ? v - r : 1;
}

// max(1, ceil(round((1 - s) * n, 9)))  — compressors.py:185-194.  Python's round(x, 9)
// is the correctly rounded decimal at 9 places; glibc printf("%.9f") is too.
int64_t top_k_count(double sparsity, int64_t n) {
  if (n < 1) return -1;
  char buf[64];
  snprintf(buf, sizeof(buf), "%.9f", (1.0 - sparsity) * (double)n);
  const double v = strtod(buf, nullptr);
  const int64_t k = (int64_t)std::ceil(v);
  return k < 1 ? 1 : k;
}

static bool spec_ok(const mc_spec* s) {
  if (!s) { set_error("null spec"); return false; }
  if (s->algorithm < 0 || s->algorithm >= MC_NUM_ALGORITHMS) { set_error("unknown algorithm id %d", s->algorithm); return false; }
  if (!(s->sparsity >= 0.0 && s->sparsity < 1.0)) { set_error("sparsity must be in [0, 1)"); return false; }
  if (s->levels < 2) { set_error("levels must be >= 2"); return false; }
  if (s->bucket_size < 1) { set_error("bucket_size must be >= 1"); return false; }
  if (s->threshold < 0) { set_error("threshold must be >= 0"); return false; }
  return true;
}

// Device payload layout (see mc_payload_header in include/mergecomp.h).
int fill_layout(const mc_spec* s, int64_t n, int64_t cap, mc_layout* L) {
  if (!spec_ok(s) || n < 1 || !L) { if (n < 1) set_error("n must be >= 1"); return MC_EINVAL; }
  memset(L, 0, sizeof(*L));
  L->n = n;
  const int64_t nb = cdiv(n, s->bucket_size);
  const int64_t sb = cdiv(n, 8);
  const int a = s->algorithm;
  if (is_sparse(a)) {
    int64_t k = top_k_count(s->sparsity, n);
    if (a == MC_THRESHOLD) k = cap > 0 ? cap : n;
    L->cap = k;
    L->n_val = k;
    L->off_idx = HDR;
    L->off_val = HDR + a16(4 * k);
    L->off_bits = L->off_val + a16(4 * k);
    L->off_codes = L->off_bits;
    L->bytes = L->off_codes;
    return MC_OK;
  }
  switch (a) {
    case MC_IDENTITY: L->n_val = n; break;
    case MC_FP16: L->n_bits = 2 * n; break;
    case MC_QSGD: L->n_val = nb; L->n_bits = sb; L->n_codes = cdiv(n * (int64_t)level_bits(s->levels), 8); break;
    case MC_SIGNSGD:
    case MC_SIGNUM: L->n_val = 1; L->n_bits = sb; break;
    case MC_EFSIGNSGD: L->n_val = nb; L->n_bits = sb; break;
    case MC_ONEBIT: L->n_val = 2 * nb; L->n_bits = sb; break;
    case MC_TERNGRAD: L->n_val = nb; L->n_bits = cdiv(2 * n, 8); break;
    case MC_INT8: L->n_val = nb; L->n_bits = n; break;
  }
  L->off_idx = HDR;
  L->off_val = HDR;
  L->off_bits = L->off_val + a16(4 * L->n_val);
  L->off_codes = L->off_bits + a16(L->n_bits);
  L->bytes = L->off_codes + a16(L->n_codes);
  return MC_OK;
}

// ---------------------------------------------------------------- numpy SeedSequence
namespace seedseq {
constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
constexpr uint32_t MIX_L = 0xca01f9ddu, MIX_R = 0x4973f715u;
__host__ __device__ inline uint32_t hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= MULT_A;
  v *= hc;
  v ^= v >> 16;
  return v;
}
__host__ __device__ inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = MIX_L * x - MIX_R * y;
  r ^= r >> 16;
  return r;
}
// SeedSequence(entropy=(root, worker, iteration, group)).generate_state(2, u64) — the same
// code on the host (mc_derive_seed) and on the device (mc_derive_keys)
__host__ __device__ inline void derive(uint64_t root, uint64_t worker, uint64_t iteration, uint64_t group,
                                       uint64_t& key_lo, uint64_t& key_hi) {
  uint32_t ent[8];
  int ne = 0;
  const uint64_t in[4] = {root, worker, iteration, group};
  for (int i = 0; i < 4; ++i) {  // _coerce_to_uint32_array: 0 -> [0], else little-endian 32-bit words
    uint64_t v = in[i];
    if (v == 0) { ent[ne++] = 0; continue; }
    while (v) { ent[ne++] = (uint32_t)(v & 0xffffffffu); v >>= 32; }
  }
  uint32_t pool[4];
  uint32_t hc = INIT_A;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < ne ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
  for (int s = 4; s < ne; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
  uint32_t st[4];
  uint32_t hb = INIT_B;
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i % 4];
    v ^= hb;
    hb *= MULT_B;
    v *= hb;
    v ^= v >> 16;
    st[i] = v;
  }
  key_lo = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
  key_hi = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
}
}  // namespace seedseq

// keys[g] = derive(root, worker, *iteration, group0 + g); then *iteration += 1 (one CTA)
__global__ void k_derive_keys(uint64_t root, uint64_t worker, uint64_t* iteration, uint64_t group0, int ngroups,
                              uint64_t* keys) {
  const uint64_t it = *iteration;
  for (int g = threadIdx.x; g < ngroups; g += blockDim.x)
    seedseq::derive(root, worker, it, group0 + (uint64_t)g, keys[2 * g], keys[2 * g + 1]);
  __syncthreads();
  if (threadIdx.x == 0) *iteration = it + 1;
}

}  // namespace mc

using namespace mc;

extern "C" {

int mc_set_sm_reserve(int32_t n) {
  return mc::g_sm_reserve.exchange(n > 0 ? n : 0);
}

int mc_abi_version(void) { return MC_ABI_VERSION; }
const char* mc_last_error(void) { return g_err; }
int64_t mc_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

int64_t mc_top_k_count(double sparsity, int64_t n) { return top_k_count(sparsity, n); }

int64_t mc_payload_bytes(const mc_spec* s, int64_t n) {
  if (!spec_ok(s) || n < 1) return MC_EINVAL;
  const int64_t nb = cdiv(n, s->bucket_size), sb = cdiv(n, 8);
  const int64_t H = 22;
  switch (s->algorithm) {
    case MC_IDENTITY: return H + 4 * n;
    case MC_FP16: return H + 2 * n;
    case MC_TOPK: case MC_RANDK: case MC_DGC_LITE: case MC_THRESHOLD: return H + 8 * top_k_count(s->sparsity, n);
    case MC_QSGD: return H + 4 * nb + sb + cdiv(n * (int64_t)level_bits(s->levels), 8);
    case MC_SIGNSGD: case MC_SIGNUM: return H + 4 + sb;
    case MC_EFSIGNSGD: return H + 4 * nb + sb;
    case MC_ONEBIT: return H + 8 * nb + sb;
    case MC_TERNGRAD: return H + 4 * nb + cdiv(2 * n, 8);
    case MC_INT8: return H + 4 * nb + n;
  }
  return MC_EINVAL;
}

int mc_payload_layout(const mc_spec* s, int64_t n, int64_t cap, mc_layout* out) { return fill_layout(s, n, cap, out); }

int64_t mc_encode_workspace_bytes(const mc_spec* s, int64_t n) {
  if (!spec_ok(s) || n < 1) return MC_EINVAL;
  switch (s->algorithm) {
    case MC_IDENTITY: case MC_FP16: return 64;
    case MC_QSGD: case MC_EFSIGNSGD: case MC_ONEBIT: case MC_TERNGRAD: case MC_INT8: return bucket_ws_bytes(s, n);
    case MC_SIGNSGD: case MC_SIGNUM: return signglobal_ws_bytes(s, n);
    default: {  // the fused single-rank path decodes its own sparse payload in this scratch
      const int64_t e = sparse_ws_bytes(s, n), d = decode_sparse_ws_bytes(n, 1);
      return e > d ? e : d;
    }
  }
}

int mc_derive_seed(uint64_t root, uint64_t worker, uint64_t iteration, uint64_t group, uint64_t* key_lo,
                   uint64_t* key_hi) {
  if (!key_lo || !key_hi) { set_error("null output"); return MC_EINVAL; }
  seedseq::derive(root, worker, iteration, group, *key_lo, *key_hi);
  return MC_OK;
}

int mc_derive_keys(uint64_t root, uint64_t worker, uint64_t* iteration, uint64_t group0, int32_t ngroups,
                   uint64_t* keys, void* stream) {
  if (!iteration || !keys || ngroups < 1) { set_error("bad mc_derive_keys arguments"); return MC_EINVAL; }
  note_launch();
  k_derive_keys<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(root, worker, iteration, group0, ngroups, keys);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

static int encode_impl(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                       uint64_t key_lo, uint64_t key_hi, void* payload, void* workspace, int64_t workspace_bytes,
                       uint32_t* err_flags, void* stream, float* out, int64_t begin = 0, int64_t count = -1,
                       int npush = 0, void* const* push_dsts = nullptr, uint32_t* const* push_flags = nullptr,
                       uint32_t epoch = 0, const uint64_t* dkey = nullptr, void* mc_dst = nullptr,
                       uint32_t* mc_flag = nullptr, const uint32_t* epoch_ptr = nullptr) {
  if (!spec_ok(s)) return MC_EINVAL;
  if (n < 1) { set_error("gradient must have at least one element"); return MC_EINVAL; }
  if (!grad || !payload || !err_flags) { set_error("null device pointer"); return MC_EINVAL; }
  if (s->error_feedback && !residual) { set_error("error feedback requires a residual buffer"); return MC_EINVAL; }
  if (s->has_momentum && !momentum) { set_error("momentum codec requires a momentum buffer"); return MC_EINVAL; }
  if (n > 0x7fffffffLL) { set_error("group length must be < 2^31"); return MC_EINVAL; }
  const int64_t need = mc_encode_workspace_bytes(s, n);
  if (workspace_bytes < need || (need > 64 && !workspace)) {
    set_error("workspace %lld < required %lld", (long long)workspace_bytes, (long long)need);
    return MC_EWORKSPACE;
  }
  EncodeArgs a{};
  a.spec = s;
  if (fill_layout(s, n, 0, &a.L) != MC_OK) return MC_EINVAL;
  a.g = grad;
  a.n = n;
  a.r = residual;
  a.m = momentum;
  a.k0 = key_lo;
  a.k1 = key_hi;
  a.payload = static_cast<uint8_t*>(payload);
  a.ws = static_cast<uint8_t*>(workspace);
  a.ws_bytes = workspace_bytes;
  a.ctx.stream = static_cast<cudaStream_t>(stream);
  a.ctx.err = err_flags;
  a.begin = begin;
  a.count = count;
  a.npush = npush;
  a.push_dsts = push_dsts;
  a.push_flags = push_flags;
  a.epoch = epoch;
  a.dkey = dkey;
  a.mc_dst = mc_dst;
  a.mc_flag = mc_flag;
  a.epoch_ptr = epoch_ptr;
  if (begin != 0 || (count >= 0 && count != n)) {  // chunked: deterministic elementwise / bucketed codecs only
    const int al = s->algorithm;
    if (begin < 0 || count < 1 || begin + count > n) { set_error("bad chunk [%lld, +%lld)", (long long)begin, (long long)count); return MC_EINVAL; }
    if (al != MC_IDENTITY && al != MC_FP16 && al != MC_EFSIGNSGD && al != MC_ONEBIT && al != MC_INT8) {
      set_error("chunked encode unsupported for algorithm %d", al);
      return MC_EINVAL;
    }
  }
  if (npush && !(s->algorithm == MC_EFSIGNSGD || s->algorithm == MC_ONEBIT || s->algorithm == MC_INT8))
    return MC_FUSED_UNSUPPORTED;  // only the pipe kernel stores into peer slots itself
  switch (s->algorithm) {
    case MC_IDENTITY: case MC_FP16: return encode_elementwise(a, out);
    case MC_QSGD: case MC_EFSIGNSGD: case MC_ONEBIT: case MC_TERNGRAD: case MC_INT8: {
      const int rc = encode_bucketed(a, out);
      if (npush) return rc;  // MC_FUSED_UNSUPPORTED: nothing launched, the caller encodes + copies
      return (rc == MC_FUSED_UNSUPPORTED && !out) ? MC_OK : rc;
    }
    case MC_SIGNSGD: case MC_SIGNUM: { const int rc = encode_sign_global(a); return rc == MC_OK && out ? MC_FUSED_UNSUPPORTED : rc; }
    case MC_TOPK: case MC_DGC_LITE: {
      if (begin != 0 || (count >= 0 && count != n)) return MC_EINVAL;
      return encode_topk(a, out);
    }
    case MC_RANDK: return encode_randk(a, out);
    case MC_THRESHOLD: return encode_threshold(a, out);
  }
  return MC_EINVAL;
}

int mc_encode(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum, uint64_t key_lo,
              uint64_t key_hi, void* payload, void* workspace, int64_t workspace_bytes, uint32_t* err_flags,
              void* stream) {
  return encode_impl(s, grad, n, residual, momentum, key_lo, key_hi, payload, workspace, workspace_bytes, err_flags,
                     stream, nullptr);
}

}  // extern "C"

namespace mc {
namespace {
struct PushArgs {
  const uint8_t* src;
  int64_t bytes;  // multiple of 16 (payload layouts are 16-byte sections)
  int ndst, nflag;
  uint8_t* dst[MC_MAX_PUSH];
  uint32_t* flag[MC_MAX_PUSH];
  uint32_t epoch;
  const uint32_t* epoch_ptr;  // device-resident epoch (graph replay) or null: `epoch`
  uint32_t* done;
  int64_t off_idx, off_val;  // sparse (threshold): only the header and the first n_idx entries move
  int sparse;
};
// Copy a finished payload into every peer slot (16-byte vectors, all CTAs), then the last
// CTA releases every rank's flag for this rank at system scope.  Threshold payloads have a
// data-dependent count inside a capacity-n buffer: the kernel reads n_idx from the device
// header and moves the header plus idx[0, n_idx) and val[0, n_idx) only — the variable-size
// exchange needs no host round trip (counts, then a padded gather).
__global__ void __launch_bounds__(256) k_push_copy(PushArgs a) {
  const uint4* src = reinterpret_cast<const uint4*>(a.src);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  if (!a.sparse) {
    const int64_t nv = a.bytes / 16;
    for (int64_t i = tid; i < nv; i += nth) {
      const uint4 v = src[i];
      for (int j = 0; j < a.ndst; ++j) reinterpret_cast<uint4*>(a.dst[j])[i] = v;
    }
  } else {
    const int64_t cnt = reinterpret_cast<const mc_payload_header*>(a.src)->n_idx;
    const int64_t nsec = (4 * cnt + 15) / 16;  // 16-byte vectors per section
    const int64_t hv = sizeof(mc_payload_header) / 16, iv = a.off_idx / 16, vv = a.off_val / 16;
    for (int64_t t = tid; t < hv + 2 * nsec; t += nth) {
      const int64_t i = t < hv ? t : (t < hv + nsec ? iv + (t - hv) : vv + (t - hv - nsec));
      const uint4 v = src[i];
      for (int j = 0; j < a.ndst; ++j) reinterpret_cast<uint4*>(a.dst[j])[i] = v;
    }
  }
  __threadfence_system();  // this thread's peer stores, system-wide, before the CTA counts in
  if (last_cta(a.done)) {
    if (threadIdx.x == 0) {
      __threadfence_system();
      const uint32_t ep = a.epoch_ptr ? *a.epoch_ptr : a.epoch;
      for (int j = 0; j < a.nflag; ++j) st_release_sys(a.flag[j], ep);
    }
  }
}
// Wait (one CTA) until every flag equals the epoch: the gathered payloads are complete.
// Bounded: a peer silent for timeout_ns sets MC_ERR_PEER_TIMEOUT and TRAPS — the context
// faults and the job fails loudly (like NCCL's watchdog abort) instead of decoding stale or
// half-written slots and losing the double-buffer invariant.
__global__ void k_push_wait(const uint32_t* flags, int n, uint32_t epoch0, const uint32_t* epoch_ptr,
                            uint64_t timeout_ns, uint32_t* err) {
  const uint32_t epoch = epoch_ptr ? *epoch_ptr : epoch0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint64_t t0 = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys(flags + i) != epoch) {
      __nanosleep(256);
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicOr(err, MC_ERR_PEER_TIMEOUT);
        __threadfence_system();
        __trap();
      }
    }
  }
  __syncthreads();
}
}  // namespace

// One store per destination from THIS device (the kernel runs where the encode kernels
// will), then a system-scope fence: the peer-exchange probe of GradSync.try_peer_exchange.
struct ProbeArgs {
  uint32_t* dst[MC_MAX_PUSH];
  int n;
  uint32_t value;
};
__global__ void k_peer_probe(ProbeArgs a) {
  for (int j = threadIdx.x; j < a.n; j += blockDim.x) st_release_sys(a.dst[j], a.value);
  __threadfence_system();
}

int launch_push_copy(const uint8_t* payload, int64_t bytes, const EncodeArgs& a, cudaStream_t st,
                     const mc_layout* sparse) {
  PushArgs pa{};
  pa.src = payload;
  pa.bytes = (bytes + 15) / 16 * 16;
  if (sparse) {
    pa.sparse = 1;
    pa.off_idx = sparse->off_idx;
    pa.off_val = sparse->off_val;
  }
  for (int j = 0; j < a.npush; ++j) {
    pa.flag[pa.nflag++] = a.push_flags[j];
    if (a.push_dsts[j] != (void*)payload) pa.dst[pa.ndst++] = static_cast<uint8_t*>(a.push_dsts[j]);
  }
  pa.epoch = a.epoch;
  pa.epoch_ptr = a.epoch_ptr;
  pa.done = reinterpret_cast<uint32_t*>(a.ws);  // the encode is complete in stream order: its scratch is free
  MC_API_CHECK(cudaMemsetAsync(pa.done, 0, 4, st));
  const unsigned g = (unsigned)imax(1, imin(cdiv(pa.bytes / 16, 256), (int64_t)sm_count() * 4));
  note_launch();
  k_push_copy<<<g, 256, 0, st>>>(pa);
  MC_LAUNCH_CHECK();
  return MC_OK;
}
}  // namespace mc

extern "C" {

static int encode_push_impl(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                            uint64_t key_lo, uint64_t key_hi, const uint64_t* dkey, void* payload, void* const* dsts,
                            uint32_t* const* flags, int32_t nranks, uint32_t epoch, const uint32_t* epoch_ptr,
                            void* workspace, int64_t workspace_bytes, uint32_t* err_flags, void* stream) {
  if (nranks < 1 || nranks > MC_MAX_PUSH || !dsts || !flags) { set_error("bad push destinations"); return MC_EINVAL; }
  const int rc = encode_impl(s, grad, n, residual, momentum, key_lo, key_hi, payload, workspace, workspace_bytes,
                             err_flags, stream, nullptr, 0, -1, nranks, dsts, flags, epoch, dkey, nullptr, nullptr,
                             epoch_ptr);
  if (rc != MC_FUSED_UNSUPPORTED) return rc;
  // this codec's kernels do not push: plain encode, then the peer copy + flags
  const int rc2 = encode_impl(s, grad, n, residual, momentum, key_lo, key_hi, payload, workspace, workspace_bytes,
                              err_flags, stream, nullptr, 0, -1, 0, nullptr, nullptr, 0, dkey);
  if (rc2 != MC_OK) return rc2;
  mc_layout L;
  if (fill_layout(s, n, 0, &L) != MC_OK) return MC_EINVAL;
  EncodeArgs a{};
  a.ws = static_cast<uint8_t*>(workspace);
  a.npush = nranks;
  a.push_dsts = dsts;
  a.push_flags = flags;
  a.epoch = epoch;
  a.epoch_ptr = epoch_ptr;
  return launch_push_copy(static_cast<const uint8_t*>(payload), L.bytes, a, static_cast<cudaStream_t>(stream),
                          s->algorithm == MC_THRESHOLD ? &L : nullptr);
}

int mc_encode_push(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                   uint64_t key_lo, uint64_t key_hi, void* payload, void* const* dsts, uint32_t* const* flags,
                   int32_t nranks, uint32_t epoch, void* workspace, int64_t workspace_bytes, uint32_t* err_flags,
                   void* stream) {
  return encode_push_impl(s, grad, n, residual, momentum, key_lo, key_hi, nullptr, payload, dsts, flags, nranks, epoch,
                          nullptr, workspace, workspace_bytes, err_flags, stream);
}

int mc_encode_push_dev(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                       const uint64_t* dkey, void* payload, void* const* dsts, uint32_t* const* flags, int32_t nranks,
                       const uint32_t* epoch, void* workspace, int64_t workspace_bytes, uint32_t* err_flags,
                       void* stream) {
  if (!epoch) { set_error("null device epoch"); return MC_EINVAL; }
  if (s && !dkey && (s->algorithm == MC_RANDK || s->algorithm == MC_QSGD || s->algorithm == MC_TERNGRAD)) {
    set_error("mc_encode_push_dev: this codec draws random numbers and needs a device key");
    return MC_EINVAL;
  }
  return encode_push_impl(s, grad, n, residual, momentum, 0, 0, dkey, payload, dsts, flags, nranks, 0, epoch,
                          workspace, workspace_bytes, err_flags, stream);
}

int mc_encode_push_mc(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                      uint64_t key_lo, uint64_t key_hi, void* payload, void* mc_slot, uint32_t* mc_flag, uint32_t epoch,
                      void* workspace, int64_t workspace_bytes, uint32_t* err_flags, void* stream) {
  if (!payload || !mc_slot || !mc_flag) { set_error("null payload / multicast slot / flag"); return MC_EINVAL; }
  void* dsts[1] = {payload};
  uint32_t* flags[1] = {mc_flag};
  const int rc = encode_impl(s, grad, n, residual, momentum, key_lo, key_hi, payload, workspace, workspace_bytes,
                             err_flags, stream, nullptr, 0, -1, 1, dsts, flags, epoch, nullptr, mc_slot, mc_flag);
  if (rc == MC_FUSED_UNSUPPORTED) {
    set_error("the multicast push needs an aligned efsignsgd / onebit / int8 group (bucket_size %% 128 == 0)");
    return MC_EINVAL;
  }
  return rc;
}

int mc_push_wait(const uint32_t* flags, int32_t nranks, uint32_t epoch, uint64_t timeout_ns, uint32_t* err_flags,
                 void* stream) {
  if (!flags || nranks < 1 || !err_flags) { set_error("bad flags"); return MC_EINVAL; }
  if (timeout_ns == 0) timeout_ns = MC_PUSH_TIMEOUT_DEFAULT_NS;
  note_launch();
  k_push_wait<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, nranks, epoch, nullptr, timeout_ns, err_flags);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int mc_push_wait_dev(const uint32_t* flags, int32_t nranks, const uint32_t* epoch, uint64_t timeout_ns,
                     uint32_t* err_flags, void* stream) {
  if (!flags || nranks < 1 || !err_flags || !epoch) { set_error("bad flags"); return MC_EINVAL; }
  if (timeout_ns == 0) timeout_ns = MC_PUSH_TIMEOUT_DEFAULT_NS;
  note_launch();
  k_push_wait<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, nranks, 0, epoch, timeout_ns, err_flags);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int mc_peer_enable(int32_t device, int32_t peer_device) {
  if (device < 0 || peer_device < 0) { set_error("bad device index"); return MC_EINVAL; }
  if (device == peer_device) return MC_OK;  // ranks sharing one GPU: plain device memory
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, device, peer_device) != cudaSuccess || !can) {
    cudaGetLastError();
    set_error("device %d cannot access device %d over P2P", device, peer_device);
    return MC_EPEER;
  }
  int prev = 0;
  MC_API_CHECK(cudaGetDevice(&prev));
  MC_API_CHECK(cudaSetDevice(device));
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); return MC_OK; }
  if (e != cudaSuccess) {
    set_error("cudaDeviceEnablePeerAccess(%d -> %d): %s", device, peer_device, cudaGetErrorString(e));
    return MC_EPEER;
  }
  return MC_OK;
}

int mc_peer_probe(uint32_t* const* dsts, int32_t n, uint32_t value, void* stream) {
  if (!dsts || n < 1 || n > MC_MAX_PUSH) { set_error("bad probe destinations"); return MC_EINVAL; }
  mc::ProbeArgs a{};
  a.n = n;
  a.value = value;
  for (int j = 0; j < n; ++j) {
    if (!dsts[j]) { set_error("null probe destination"); return MC_EINVAL; }
    a.dst[j] = dsts[j];
  }
  mc::note_launch();
  mc::k_peer_probe<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int mc_encode_range(const mc_spec* s, const float* grad, int64_t n, int64_t begin, int64_t count, double* residual,
                    float* momentum, uint64_t key_lo, uint64_t key_hi, void* payload, void* workspace,
                    int64_t workspace_bytes, float* out, uint32_t* err_flags, void* stream) {
  const int rc = encode_impl(s, grad, n, residual, momentum, key_lo, key_hi, payload, workspace, workspace_bytes,
                             err_flags, stream, out, begin, count);
  if (rc == MC_FUSED_UNSUPPORTED) { set_error("fused decode unavailable on this path"); return MC_EINVAL; }
  return rc;
}

int mc_encode_dk(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                 const uint64_t* dkey, void* payload, void* workspace, int64_t workspace_bytes, uint32_t* err_flags,
                 void* stream) {
  if (!dkey) { set_error("null device key"); return MC_EINVAL; }
  return encode_impl(s, grad, n, residual, momentum, 0, 0, payload, workspace, workspace_bytes, err_flags, stream,
                     nullptr, 0, -1, 0, nullptr, nullptr, 0, dkey);
}

int mc_encode_decode_dk(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                        const uint64_t* dkey, void* payload, void* workspace, int64_t workspace_bytes, float* out,
                        uint32_t* err_flags, void* stream) {
  if (!out || !dkey) { set_error("null output or device key"); return MC_EINVAL; }
  const int rc = encode_impl(s, grad, n, residual, momentum, 0, 0, payload, workspace, workspace_bytes, err_flags,
                             stream, out, 0, -1, 0, nullptr, nullptr, 0, dkey);
  if (rc != MC_FUSED_UNSUPPORTED) return rc;
  return mc_decode_mean_ws(s, payload, 0, 1, n, out, workspace, workspace_bytes, err_flags, stream);
}

int mc_encode_decode(const mc_spec* s, const float* grad, int64_t n, double* residual, float* momentum,
                     uint64_t key_lo, uint64_t key_hi, void* payload, void* workspace, int64_t workspace_bytes,
                     float* out, uint32_t* err_flags, void* stream) {
  if (!out) { set_error("null output"); return MC_EINVAL; }
  const int rc = encode_impl(s, grad, n, residual, momentum, key_lo, key_hi, payload, workspace, workspace_bytes,
                             err_flags, stream, out);
  if (rc != MC_FUSED_UNSUPPORTED) return rc;
  // two-pass codecs: decode the own payload; the encode's scratch is free again in stream order
  return mc_decode_mean_ws(s, payload, 0, 1, n, out, workspace, workspace_bytes, err_flags, stream);
}

int64_t mc_decode_workspace_bytes(const mc_spec* s, int64_t n, int32_t nranks) {
  if (!spec_ok(s) || n < 1 || nranks < 1) return MC_EINVAL;
  return is_sparse(s->algorithm) ? decode_sparse_ws_bytes(n, nranks) : 0;
}

int mc_decode_mean_ws(const mc_spec* s, const void* payloads, int64_t stride_bytes, int32_t nranks, int64_t n,
                      float* out, void* workspace, int64_t workspace_bytes, uint32_t* err_flags, void* stream) {
  if (!spec_ok(s)) return MC_EINVAL;
  if (n < 1 || nranks < 1 || !payloads || !out || !err_flags) { set_error("bad decode arguments"); return MC_EINVAL; }
  if (nranks > 1 && stride_bytes < 32) { set_error("stride too small"); return MC_EINVAL; }
  mc_layout L;
  if (fill_layout(s, n, 0, &L) != MC_OK) return MC_EINVAL;
  Ctx c{static_cast<cudaStream_t>(stream), err_flags};
  const uint8_t* base = static_cast<const uint8_t*>(payloads);
  if (is_sparse(s->algorithm)) return decode_mean_sparse(s, L, base, stride_bytes, nranks, out, c, workspace, workspace_bytes);
  return decode_mean_dense(s, L, base, stride_bytes, nranks, out, c);
}

int mc_decode_mean(const mc_spec* s, const void* payloads, int64_t stride_bytes, int32_t nranks, int64_t n, float* out,
                   uint32_t* err_flags, void* stream) {
  return mc_decode_mean_ws(s, payloads, stride_bytes, nranks, n, out, nullptr, 0, err_flags, stream);
}

}  // extern "C"

// ---------------------------------------------------------------- merge stage + serialize
namespace mc {
namespace {

// Merge stage (K1 / K11 of SURVEY.md §2.1): per-layer gradients <-> one fused buffer in list
// order.  Work is split on the host into CTA chunks of PACK_CHUNK elements of ONE tensor
// (blk0[i] = first chunk of tensor i), so a CTA finds its tensor with one uniform binary
// search over the parameter table and then streams a contiguous run: 128-bit loads and
// stores whenever source and destination share their 16-byte phase (a scalar head aligns
// them), scalar otherwise.  Pure HBM copy: 8 B/element.
constexpr int PACK_MAX = 512;    // tensors per launch (parameter table, ~14 KB)
constexpr int PACK_CHUNK = 8192;  // elements per CTA
struct PackArgs {
  const float* src[PACK_MAX];
  float* dst[PACK_MAX];
  int64_t off[PACK_MAX + 1];  // element offset of tensor i inside the fused buffer
  int32_t blk0[PACK_MAX + 1];  // first CTA chunk of tensor i
  int count;
  int to_fused;  // 1: pack (tensors -> fused), 0: unpack (fused -> tensors)
  float* fused;
  const float* cfused;
};

__global__ void __launch_bounds__(256) k_pack(const __grid_constant__ PackArgs a) {
  const int b = blockIdx.x;
  int lo = 0, hi = a.count - 1;  // tensor of this chunk: largest i with blk0[i] <= b
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.blk0[mid] <= b) lo = mid; else hi = mid - 1;
  }
  const int64_t numel = a.off[lo + 1] - a.off[lo];
  const int64_t j0 = (int64_t)(b - a.blk0[lo]) * PACK_CHUNK;
  const int64_t len = imin(PACK_CHUNK, numel - j0);
  const float* src = a.to_fused ? a.src[lo] + j0 : a.cfused + a.off[lo] + j0;
  float* dst = a.to_fused ? a.fused + a.off[lo] + j0 : a.dst[lo] + j0;
  const uintptr_t ps = (uintptr_t)src & 15, pd = (uintptr_t)dst & 15;
  int64_t head = 0;
  if (ps == pd) head = imin(len, (int64_t)(((16 - ps) & 15) >> 2));  // same phase: align both
  else head = len;                                                    // different phase: scalar
  for (int64_t e = threadIdx.x; e < head; e += blockDim.x) dst[e] = src[e];
  const int64_t nv = (len - head) >> 2;
  const float4* s4 = reinterpret_cast<const float4*>(src + head);
  float4* d4 = reinterpret_cast<float4*>(dst + head);
  for (int64_t v = threadIdx.x; v < nv; v += blockDim.x) d4[v] = __ldcs(s4 + v);
  for (int64_t e = head + 4 * nv + threadIdx.x; e < len; e += blockDim.x) dst[e] = src[e];
}

int pack_impl(const float* const* srcs, float* const* dsts, const int64_t* numels, int32_t count, float* fused,
              const float* cfused, int to_fused, cudaStream_t st) {
  if (count < 0 || !numels || (count > 0 && (to_fused ? !srcs : !dsts))) { set_error("bad pack arguments"); return MC_EINVAL; }
  if (to_fused ? !fused : !cfused) { set_error("null fused buffer"); return MC_EINVAL; }
  int64_t base = 0;
  for (int32_t i0 = 0; i0 < count; i0 += PACK_MAX) {
    PackArgs a{};
    a.count = (int)imin(PACK_MAX, count - i0);
    a.to_fused = to_fused;
    a.off[0] = 0;
    a.blk0[0] = 0;
    for (int i = 0; i < a.count; ++i) {
      const int64_t m = numels[i0 + i];
      if (m < 0) { set_error("negative numel"); return MC_EINVAL; }
      if (m > 0 && (to_fused ? !srcs[i0 + i] : !dsts[i0 + i])) { set_error("null tensor pointer"); return MC_EINVAL; }
      if (to_fused) a.src[i] = srcs[i0 + i]; else a.dst[i] = dsts[i0 + i];
      a.off[i + 1] = a.off[i] + m;
      const int64_t nb = a.blk0[i] + cdiv(m, PACK_CHUNK);
      if (nb > 0x7fffffff) { set_error("merge stage too large for one launch"); return MC_EINVAL; }
      a.blk0[i + 1] = (int32_t)nb;
    }
    a.fused = fused ? fused + base : nullptr;
    a.cfused = cfused ? cfused + base : nullptr;
    if (a.blk0[a.count] > 0) {
      note_launch(); k_pack<<<(unsigned)a.blk0[a.count], 256, 0, st>>>(a);
      MC_LAUNCH_CHECK();
    }
    base += a.off[a.count];
  }
  return MC_OK;
}

struct SerArgs {
  uint8_t header[24];
  const uint8_t* src[4];
  int64_t len[4];
  int64_t start[5];  // output offsets of the 4 sections (start[0] = 22)
  uint8_t* out;
};

__global__ void k_serialize(SerArgs a) {
  const int64_t total = a.start[4];
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    if (o < 22) { a.out[o] = a.header[o]; continue; }
    int s = 0;
    while (s < 3 && o >= a.start[s + 1]) ++s;
    a.out[o] = a.src[s][o - a.start[s]];
  }
}

// Inverse of k_serialize: canonical bytes (22-byte header + packed sections) -> the
// aligned device layout; thread 0..31 write the 32-byte mc_payload_header.
struct DeserArgs {
  mc_payload_header h;
  const uint8_t* in;
  uint8_t* dst[4];
  int64_t len[4];
  int64_t start[5];  // input offsets of the 4 sections (start[0] = 22)
  uint8_t* payload;
};

__global__ void k_deserialize(DeserArgs a) {
  const int64_t total = a.start[4];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid < (int64_t)sizeof(mc_payload_header)) a.payload[tid] = reinterpret_cast<const uint8_t*>(&a.h)[tid];
  for (int64_t o = 22 + tid; o < total; o += (int64_t)gridDim.x * blockDim.x) {
    int s = 0;
    while (s < 3 && o >= a.start[s + 1]) ++s;
    a.dst[s][o - a.start[s]] = a.in[o];
  }
}

}  // namespace
}  // namespace mc

extern "C" {

int mc_pack(const float* const* srcs, const int64_t* numels, int32_t count, float* fused, void* stream) {
  if (!fused && count > 0) { set_error("null fused buffer"); return MC_EINVAL; }
  return mc::pack_impl(srcs, nullptr, numels, count, fused, nullptr, 1, static_cast<cudaStream_t>(stream));
}

int mc_unpack(const float* fused, float* const* dsts, const int64_t* numels, int32_t count, void* stream) {
  if (!fused && count > 0) { set_error("null fused buffer"); return MC_EINVAL; }
  return mc::pack_impl(nullptr, dsts, numels, count, nullptr, fused, 0, static_cast<cudaStream_t>(stream));
}

int mc_serialize(const mc_spec* s, const void* payload, int64_t n, void* out, int64_t out_cap, int64_t* out_len,
                 void* stream) {
  mc_layout L;
  if (fill_layout(s, n, 0, &L) != MC_OK) return MC_EINVAL;
  if (!payload || !out || !out_len) { set_error("null pointer"); return MC_EINVAL; }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  mc_payload_header h;
  if (cudaMemcpyAsync(&h, payload, sizeof(h), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("reading payload header failed");
    return MC_ECUDA;
  }
  if ((int)h.algorithm != s->algorithm || h.original_len != (uint64_t)n) { set_error("payload header mismatch"); return MC_EINVAL; }
  const uint8_t* p = static_cast<const uint8_t*>(payload);
  SerArgs a{};
  const int64_t nidx = h.n_idx, nval = h.n_val;
  const bool sparse = is_sparse(s->algorithm);
  a.src[0] = p + HDR;
  a.len[0] = 4 * nidx;
  a.src[1] = sparse ? p + HDR + a16(4 * (int64_t)h.cap) : p + L.off_val;
  a.len[1] = 4 * nval;
  a.src[2] = p + L.off_bits;
  a.len[2] = sparse ? 0 : L.n_bits;
  a.src[3] = p + L.off_codes;
  a.len[3] = sparse ? 0 : L.n_codes;
  a.start[0] = 22;
  for (int i = 0; i < 4; ++i) a.start[i + 1] = a.start[i] + a.len[i];
  const uint32_t nbits = (uint32_t)(a.len[2] + a.len[3]);
  // "<BBQIII": algo u8, flags u8, original_len u64, n_idx u32, n_val u32, n_bits u32
  a.header[0] = (uint8_t)h.algorithm;
  a.header[1] = (uint8_t)h.flags;
  memcpy(a.header + 2, &h.original_len, 8);
  const uint32_t ni = (uint32_t)nidx, nv = (uint32_t)nval;
  memcpy(a.header + 10, &ni, 4);
  memcpy(a.header + 14, &nv, 4);
  memcpy(a.header + 18, &nbits, 4);
  a.out = static_cast<uint8_t*>(out);
  *out_len = a.start[4];
  if (out_cap < a.start[4]) { set_error("serialize buffer too small (%lld < %lld)", (long long)out_cap, (long long)a.start[4]); return MC_EINVAL; }
  const unsigned grid = (unsigned)imax(1, imin(cdiv(a.start[4], 256), 4096));
  note_launch(); k_serialize<<<grid, 256, 0, st>>>(a);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int mc_deserialize(const mc_spec* s, const void* data, int64_t len, void* payload, int64_t payload_cap,
                   int64_t* n_out, void* stream) {
  using namespace mc;
  if (!spec_ok(s)) return MC_EINVAL;
  if (!data || !payload || !n_out) { set_error("null pointer"); return MC_EINVAL; }
  if (len < 22) { set_error("payload shorter than header"); return MC_EINVAL; }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t raw[22];
  if (cudaMemcpyAsync(raw, data, 22, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("reading payload header failed");
    return MC_ECUDA;
  }
  // "<BBQIII" (compressors.py:53, 623-645)
  uint64_t n;
  uint32_t nidx, nval, nbits;
  memcpy(&n, raw + 2, 8);
  memcpy(&nidx, raw + 10, 4);
  memcpy(&nval, raw + 14, 4);
  memcpy(&nbits, raw + 18, 4);
  const int algo = raw[0];
  if (algo >= MC_NUM_ALGORITHMS) { set_error("unknown algorithm id %d", algo); return MC_EINVAL; }
  const int64_t expect = 22 + 4 * (int64_t)nidx + 4 * (int64_t)nval + (int64_t)nbits;
  if (len != expect) { set_error("payload length %lld does not match header (%lld)", (long long)len, (long long)expect); return MC_EINVAL; }
  if (algo != s->algorithm) { set_error("payload algorithm id %d does not match spec id %d", algo, s->algorithm); return MC_EINVAL; }
  if (n < 1) { set_error("corrupt payload: zero length"); return MC_EINVAL; }
  const bool sparse = is_sparse(algo);
  mc_layout L;
  if (fill_layout(s, (int64_t)n, sparse ? (int64_t)(nidx > 0 ? nidx : 1) : 0, &L) != MC_OK) return MC_EINVAL;
  DeserArgs a{};
  uint8_t* p = static_cast<uint8_t*>(payload);
  if (sparse) {
    if (nidx != nval) { set_error("corrupt payload: index/value length mismatch"); return MC_EINVAL; }
    if (nbits != 0) { set_error("corrupt payload: sparsifier payload carries bits"); return MC_EINVAL; }
    if (algo != MC_THRESHOLD && (int64_t)nidx != L.cap) { set_error("corrupt payload: expected %lld indices", (long long)L.cap); return MC_EINVAL; }
    L.cap = nidx;
    L.n_val = nidx;
    L.off_val = HDR + a16(4 * (int64_t)nidx);
    L.bytes = L.off_val + a16(4 * (int64_t)nidx);
    a.dst[0] = p + HDR;
    a.dst[1] = p + L.off_val;
  } else {
    if (nidx != 0) { set_error("corrupt payload: dense payload carries indices"); return MC_EINVAL; }
    if ((int64_t)nval != L.n_val) { set_error("corrupt payload: value count %u, expected %lld", nval, (long long)L.n_val); return MC_EINVAL; }
    if ((int64_t)nbits != L.n_bits + L.n_codes) { set_error("corrupt payload: bit buffer length %u, expected %lld", nbits, (long long)(L.n_bits + L.n_codes)); return MC_EINVAL; }
    a.dst[0] = p + HDR;
    a.dst[1] = p + L.off_val;
    a.dst[2] = p + L.off_bits;
    a.dst[3] = p + L.off_codes;
  }
  if (payload_cap < L.bytes) { set_error("payload buffer too small (%lld < %lld)", (long long)payload_cap, (long long)L.bytes); return MC_EINVAL; }
  a.len[0] = 4 * (int64_t)nidx;
  a.len[1] = 4 * (int64_t)nval;
  a.len[2] = sparse ? 0 : L.n_bits;
  a.len[3] = sparse ? 0 : L.n_codes;
  a.start[0] = 22;
  for (int i = 0; i < 4; ++i) a.start[i + 1] = a.start[i] + a.len[i];
  a.h.algorithm = (uint32_t)algo;
  a.h.flags = raw[1];
  a.h.original_len = n;
  a.h.n_idx = nidx;
  a.h.n_val = nval;
  a.h.n_bits = nbits;
  a.h.cap = sparse ? nidx : 0;
  a.in = static_cast<const uint8_t*>(data);
  a.payload = p;
  *n_out = (int64_t)n;
  const unsigned grid = (unsigned)imax(1, imin(cdiv(len, 256), 4096));
  note_launch(); k_deserialize<<<grid, 256, 0, st>>>(a);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

}  // extern "C"
