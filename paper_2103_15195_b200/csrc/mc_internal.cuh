// mc_internal.cuh — shared device machinery of the sm_100a MergeComp kernels.
//
// Numerics contract: every float operation that the reference
// performs in numpy is reproduced with an explicitly rounded intrinsic
// (__fadd_rn/__fmul_rn/__fdiv_rn/__dadd_rn/...), the library is compiled with
// --fmad=false and without fast-math, so results are bit-identical to the
// numpy expressions cited at each use.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/mergecomp.h"

namespace mc {

constexpr unsigned FULL = 0xffffffffu;
constexpr int HDR = 32;  // sizeof(mc_payload_header)

__host__ __device__ inline int64_t a16(int64_t x) { return (x + 15) & ~int64_t(15); }
__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ inline int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ inline int level_bits(int levels) {
  int v = levels - 1, b = 0;
  while (v) { ++b; v >>= 1; }
  return b < 1 ? 1 : b;
}
inline bool is_sparse(int a) { return a == MC_TOPK || a == MC_RANDK || a == MC_DGC_LITE || a == MC_THRESHOLD; }

int64_t top_k_count(double sparsity, int64_t n);
int fill_layout(const mc_spec* s, int64_t n, int64_t cap, mc_layout* L);
int sm_count();  // of the current device (cached per device)

// Dynamic shared memory above 48 KB is opted into per kernel AND per device: `mask` is the
// call site's own set of devices already configured (one static per kernel instantiation),
// so a process driving several GPUs configures each of them.
template <class F>
inline cudaError_t smem_optin(std::atomic<uint64_t>& mask, F* kernel, int bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_release);
  return e;
}
void set_error(const char* fmt, ...);
void note_launch();  // counts kernel launches (mc_kernel_launches)

// --------------------------------------------------------------------------------------------
// Per-call launch context.
struct Ctx {
  cudaStream_t stream;
  uint32_t* err;
};

#define MC_LAUNCH_CHECK()                                                           \
  do {                                                                              \
    cudaError_t e_ = cudaGetLastError();                                            \
    if (e_ != cudaSuccess) {                                                        \
      ::mc::set_error("CUDA launch failed: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return MC_ECUDA;                                                              \
    }                                                                               \
  } while (0)

#define MC_API_CHECK(call)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      ::mc::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
      return MC_ECUDA;                                                                     \
    }                                                                                      \
  } while (0)

// --------------------------------------------------------------------------------------------
// Philox4x64-10, counter = (block + 1, 0, 0, 0): numpy's Philox bit generator
// (Random123 round function).  Uniform double = (w >> 11) * 2^-53
// (compared without forming it: u53_below in mc_bucket.cu).
struct Philox {
  uint64_t k0, k1;
  __device__ __forceinline__ void block(uint64_t blk, uint64_t out[4]) const {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
    uint64_t c0 = blk + 1, c1 = 0, c2 = 0, c3 = 0, a = k0, b = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r) { a += W0; b += W1; }
      const uint64_t lo0 = M0 * c0, hi0 = __umul64hi(M0, c0);
      const uint64_t lo1 = M1 * c2, hi1 = __umul64hi(M1, c2);
      c0 = hi1 ^ c1 ^ a; c1 = lo1; c2 = hi0 ^ c3 ^ b; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
  }
};

// The same generator with its round keys (a_r, b_r) = (k0 + r W0, k1 + r W1) computed once on
// the host and passed in the kernel parameters: the rounds then take the keys as constant-bank
// operands (LOP3 ..., c[0x0][...]) instead of re-deriving the schedule for every block.
struct PhiloxKS {
  uint64_t a[10], b[10];
  uint64_t x1, x2;  // hi(M0 a0) ^ b1 and lo(M0 a0) ^ b2: round 1's M0 product is a key constant
  __host__ __device__ static PhiloxKS make(uint64_t k0, uint64_t k1) {
    PhiloxKS ks;
    for (int r = 0; r < 10; ++r) {
      ks.a[r] = k0 + (uint64_t)r * 0x9E3779B97F4A7C15ull;
      ks.b[r] = k1 + (uint64_t)r * 0xBB67AE8584CAA73Bull;
    }
#ifdef __CUDA_ARCH__
    const uint64_t ulo = 0xD2E7470EE14C6C93ull * ks.a[0], uhi = __umul64hi(0xD2E7470EE14C6C93ull, ks.a[0]);
#else
    const unsigned __int128 u = (unsigned __int128)0xD2E7470EE14C6C93ull * ks.a[0];
    const uint64_t ulo = (uint64_t)u, uhi = (uint64_t)(u >> 64);
#endif
    ks.x1 = uhi ^ ks.b[1];
    ks.x2 = ulo ^ ks.b[2];
    return ks;
  }
  // One block whose counter ctr = blk + 1 fits 32 bits (streams under 2^34 draws).  Round 0
  // runs on (ctr, 0, 0, 0): a 64 x 32-bit product and no M1 product; round 1 enters with
  // c0 = a0 and c1 = 0, so its M0 product is the key constant folded into x1 / x2 — 70
  // 32-bit wide multiplies per block instead of 80.  Bit-identical to block(ctr - 1).
  __device__ __forceinline__ void block32(uint32_t ctr, uint64_t out[4]) const {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t p0 = (uint64_t)(uint32_t)M0 * ctr, p1 = (uint64_t)(uint32_t)(M0 >> 32) * ctr;
    const uint64_t t = (p0 >> 32) + (uint32_t)p1;
    const uint64_t lo = (t << 32) | (uint32_t)p0, hi = (p1 >> 32) + (t >> 32);  // M0 * ctr
    uint64_t c2 = hi ^ b[0];                                                      // round 0
    uint64_t c0 = __umul64hi(M1, c2) ^ a[1], c1 = M1 * c2, c3;                    // round 1
    c2 = lo ^ x1;
    {                                                                             // round 2
      const uint64_t lo0 = M0 * c0, hi0 = __umul64hi(M0, c0);
      const uint64_t lo1 = M1 * c2, hi1 = __umul64hi(M1, c2);
      c0 = hi1 ^ c1 ^ a[2]; c1 = lo1; c2 = hi0 ^ x2; c3 = lo0;
    }
#pragma unroll
    for (int r = 3; r < 10; ++r) {
      const uint64_t lo0 = M0 * c0, hi0 = __umul64hi(M0, c0);
      const uint64_t lo1 = M1 * c2, hi1 = __umul64hi(M1, c2);
      c0 = hi1 ^ c1 ^ a[r]; c1 = lo1; c2 = hi0 ^ c3 ^ b[r]; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
  }
  __device__ __forceinline__ void block(uint64_t blk, uint64_t out[4]) const {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    uint64_t c0 = blk + 1, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      const uint64_t lo0 = M0 * c0, hi0 = __umul64hi(M0, c0);
      const uint64_t lo1 = M1 * c2, hi1 = __umul64hi(M1, c2);
      c0 = hi1 ^ c1 ^ a[r]; c1 = lo1; c2 = hi0 ^ c3 ^ b[r]; c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
  }
  // J independent blocks blk0 + j*stride, rounds interleaved (J-way ILP on the IMAD chain)
  template <int J>
  __device__ __forceinline__ void blocks(uint64_t blk0, uint64_t stride, uint64_t (&out)[J][4]) const {
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    uint64_t c0[J], c1[J], c2[J], c3[J];
#pragma unroll
    for (int j = 0; j < J; ++j) { c0[j] = blk0 + (uint64_t)j * stride + 1; c1[j] = c2[j] = c3[j] = 0; }
#pragma unroll
    for (int r = 0; r < 10; ++r)
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const uint64_t lo0 = M0 * c0[j], hi0 = __umul64hi(M0, c0[j]);
        const uint64_t lo1 = M1 * c2[j], hi1 = __umul64hi(M1, c2[j]);
        c0[j] = hi1 ^ c1[j] ^ a[r]; c1[j] = lo1; c2[j] = hi0 ^ c3[j] ^ b[r]; c3[j] = lo0;
      }
#pragma unroll
    for (int j = 0; j < J; ++j) { out[j][0] = c0[j]; out[j][1] = c1[j]; out[j][2] = c2[j]; out[j][3] = c3[j]; }
  }
};

// --------------------------------------------------------------------------------------------
// numpy float32 pairwise summation (umath loops_utils pairwise_sum):
//   n < 8   : s = -0; s += a[i] sequentially
//   n <= 128: 8 strided accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail
//   else    : m = n/2 - (n/2)%8 ; P(a[:m]) + P(a[m:])
// The ufunc reduce adds the result to a +0 identity, which callers apply.
// Warp-cooperative, iterative post-order walk (identical control flow in all lanes);
// `get(q)` returns element q of the sequence.  Result is valid in every lane.
template <class Get>
__device__ float warp_pairwise(const Get& get, int64_t L) {
  const int lane = threadIdx.x & 31;
  int64_t st_off[48], st_len[48];  // node stack; len < 0 marks "combine"
  float vals[24];
  int sp = 0, vp = 0;
  st_off[sp] = 0; st_len[sp] = L; ++sp;
  while (sp) {
    --sp;
    const int64_t off = st_off[sp], len = st_len[sp];
    if (len < 0) {
      const float b = vals[--vp], a = vals[--vp];
      vals[vp++] = __fadd_rn(a, b);
      continue;
    }
    if (len > 128) {
      int64_t m = len / 2;
      m -= m % 8;
      st_off[sp] = 0; st_len[sp] = -1; ++sp;        // combine after both children
      st_off[sp] = off + m; st_len[sp] = len - m; ++sp;
      st_off[sp] = off; st_len[sp] = m; ++sp;       // left child processed first
      continue;
    }
    float res;
    if (len < 8) {
      float s = -0.0f;
      if (lane == 0)
        for (int64_t q = 0; q < len; ++q) s = __fadd_rn(s, get(off + q));
      res = __shfl_sync(FULL, s, 0);
    } else {
      const int64_t body = len - (len % 8);
      float r = 0.0f;
      if (lane < 8) {
        r = get(off + lane);
        for (int64_t i = 8; i < body; i += 8) r = __fadd_rn(r, get(off + i + lane));
      }
      r = __fadd_rn(r, __shfl_xor_sync(FULL, r, 1));
      r = __fadd_rn(r, __shfl_xor_sync(FULL, r, 2));
      r = __fadd_rn(r, __shfl_xor_sync(FULL, r, 4));
      float s = r;
      if (lane == 0)
        for (int64_t q = body; q < len; ++q) s = __fadd_rn(s, get(off + q));
      res = __shfl_sync(FULL, s, 0);
    }
    vals[vp++] = res;
  }
  return vals[0];
}

// Bounded-depth variant for L <= 128 * 2^D (D <= 4 covers L <= 1024 with <= 9 leaves): the
// leaves of the numpy tree are enumerated by a compile-time-unrolled recursion (warp
// uniform), summed 4 at a time by 8-lane groups (all 32 lanes busy), and recombined by
// the same recursion.  Bitwise identical to warp_pairwise.
namespace pw {
template <int D>
__device__ __forceinline__ void collect(int off, int len, int& cnt, int& my_off, int& my_len) {
  if (D == 0 || len <= 128) {
    if ((int)(threadIdx.x & 31) == cnt) { my_off = off; my_len = len; }
    ++cnt;
    return;
  }
  int m = len / 2;
  m -= m % 8;
  collect<(D > 0 ? D - 1 : 0)>(off, m, cnt, my_off, my_len);
  collect<(D > 0 ? D - 1 : 0)>(off + m, len - m, cnt, my_off, my_len);
}
template <int D>
__device__ __forceinline__ float combine(int len, int& cnt, float leafv) {
  if (D == 0 || len <= 128) return __shfl_sync(0xffffffffu, leafv, cnt++);
  int m = len / 2;
  m -= m % 8;
  const float a = combine<(D > 0 ? D - 1 : 0)>(m, cnt, leafv);
  const float b = combine<(D > 0 ? D - 1 : 0)>(len - m, cnt, leafv);
  return __fadd_rn(a, b);
}
}  // namespace pw

template <int D, class Get>
__device__ __forceinline__ float warp_pairwise_small(const Get& get, int L) {
  const int lane = threadIdx.x & 31;
  if (L < 8) {  // single short leaf: sequential from -0.0
    float s = -0.0f;
    if (lane == 0)
      for (int q = 0; q < L; ++q) s = __fadd_rn(s, get(q));
    return __shfl_sync(FULL, s, 0);
  }
  int nleaf = 0, my_off = 0, my_len = 0;
  pw::collect<D>(0, L, nleaf, my_off, my_len);
  float leafv = 0.0f;  // lane k ends up holding leaf k's sum
  for (int base = 0; base < nleaf; base += 4) {
    const int g = lane >> 3, j = lane & 7, leaf = base + g;
    const int off = __shfl_sync(FULL, my_off, leaf & 31), len = __shfl_sync(FULL, my_len, leaf & 31);
    const bool act = leaf < nleaf;
    const int body = act ? len - (len % 8) : 0;
    float r = act ? get(off + j) : 0.0f;
#pragma unroll
    for (int t = 1; t < 16; ++t)
      if (8 * t < body) r = __fadd_rn(r, get(off + 8 * t + j));
    r = __fadd_rn(r, __shfl_xor_sync(FULL, r, 1));
    r = __fadd_rn(r, __shfl_xor_sync(FULL, r, 2));
    r = __fadd_rn(r, __shfl_xor_sync(FULL, r, 4));
    if (act && j == 0)
      for (int q = body; q < len; ++q) r = __fadd_rn(r, get(off + q));
#pragma unroll
    for (int gg = 0; gg < 4; ++gg) {
      const float v = __shfl_sync(FULL, r, 8 * gg);
      if (lane == base + gg) leafv = v;
    }
  }
  int cnt = 0;
  return pw::combine<D>(L, cnt, leafv);
}

__device__ __forceinline__ int pad32(int q) { return q + 8 * (q >> 5); }

// warp_pairwise_small over the pad32() layout (q + 8 * (q >> 5)) with the leaf reads addressed from four
// per-lane bases: lane j of a leaf group reads q = o + 8t (o = leaf offset + j, leaf offsets
// are multiples of 8), whose padded position is pad32(o) + 8t + 8*((k + t) >> 2) with
// k = (o >> 3) & 3; for t = 4u + r that is B_r + 8t + 8u, B_r = pad32(o) + 8*((k + r) >> 2),
// so every unrolled read is one LDS with an immediate offset.  Same sums, same order.
template <int D>
__device__ __forceinline__ float pairwise_pad32(const float* a, int L) {
  const int lane = threadIdx.x & 31;
  if (L < 8) {
    float s = -0.0f;
    if (lane == 0)
      for (int q = 0; q < L; ++q) s = __fadd_rn(s, a[pad32(q)]);
    return __shfl_sync(FULL, s, 0);
  }
  int nleaf = 0, my_off = 0, my_len = 0;
  pw::collect<D>(0, L, nleaf, my_off, my_len);
  float leafv = 0.0f;
  for (int base = 0; base < nleaf; base += 4) {
    const int g = lane >> 3, j = lane & 7, leaf = base + g;
    const int off = __shfl_sync(FULL, my_off, leaf & 31), len = __shfl_sync(FULL, my_len, leaf & 31);
    const bool act = leaf < nleaf;
    const int body = act ? len - (len % 8) : 0;
    const int o = off + j, k = (o >> 3) & 3;
    const float* B[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) B[r] = a + pad32(o) + 8 * ((k + r) >> 2);
    float v = act ? B[0][0] : 0.0f;
    if (L > 128) {  // leaves of a split are >= 64 long: rows 1..7 always exist (inactive lanes
                    // add in-bounds garbage nobody reads)
#pragma unroll
      for (int t = 1; t < 8; ++t) v = __fadd_rn(v, B[t & 3][8 * t + 8 * (t >> 2)]);
#pragma unroll
      for (int t = 8; t < 16; ++t)
        if (8 * t < body) v = __fadd_rn(v, B[t & 3][8 * t + 8 * (t >> 2)]);
    } else {
#pragma unroll
      for (int t = 1; t < 16; ++t)
        if (8 * t < body) v = __fadd_rn(v, B[t & 3][8 * t + 8 * (t >> 2)]);
    }
    v = __fadd_rn(v, __shfl_xor_sync(FULL, v, 1));
    v = __fadd_rn(v, __shfl_xor_sync(FULL, v, 2));
    v = __fadd_rn(v, __shfl_xor_sync(FULL, v, 4));
    if (act && j == 0)
      for (int q = body; q < len; ++q) v = __fadd_rn(v, a[pad32(off + q)]);
#pragma unroll
    for (int gg = 0; gg < 4; ++gg) {
      const float w = __shfl_sync(FULL, v, 8 * gg);
      if (lane == base + gg) leafv = w;
    }
  }
  int cnt = 0;
  return pw::combine<D>(L, cnt, leafv);
}

// numpy float32 mean of a sequence with a known pairwise sum:  f32( f64(0 + P) / n ).
__device__ __forceinline__ float np_mean(float pairwise_sum, int64_t n) {
  const float s = __fadd_rn(0.0f, pairwise_sum);
  return __double2float_rn(__ddiv_rn((double)s, (double)n));
}

// --------------------------------------------------------------------------------------------
// Decoupled look-back prefix scan across blocks (one 64-bit status word per block:
// 2 flag bits | 62-bit value).  Blocks take tickets in launch order so every
// predecessor is resident or finished — forward progress is guaranteed.
constexpr uint64_t LB_AGG = 1ull << 62, LB_PRE = 2ull << 62, LB_MASK = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) {
  return *reinterpret_cast<const volatile uint64_t*>(p);
}
// Status words are published with an atomic exchange: performed at L2, visible to every
// polling CTA at once without a membar (which would also drain this warp's output stores).
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) {
  atomicExch(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

// Called by warp 0 of a block with its aggregate; returns the exclusive prefix in all lanes.
__device__ __forceinline__ uint64_t lookback_warp(uint64_t* status, int64_t bid, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (bid == 0) {
    if (lane == 0) { st_volatile(&status[0], LB_PRE | agg); }
    return 0;
  }
  // Flag and value travel in one 64-bit word published atomically at L2, so a reader sees
  // either nothing or a complete entry, and no other data is published through it.
  if (lane == 0) { st_volatile(&status[bid], LB_AGG | agg); }
  // Each step inspects a window of 32 lanes x 4 predecessors (newest first), so a block
  // that has to walk back over many aggregate-only entries (thousands of CTAs in flight)
  // pays few dependent L2 round trips.
  uint64_t prefix = 0;
  int64_t j = bid - 1;
  while (true) {
    uint64_t s[4];
    // issue the 4 loads back to back (one round trip), then re-poll only unpublished ones
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t idx = j - 4 * lane - q;
      s[q] = idx >= 0 ? ld_volatile(&status[idx]) : LB_PRE;  // before block 0: empty prefix
    }
    while (true) {
      bool ready = true;
#pragma unroll
      for (int q = 0; q < 4; ++q) ready &= (s[q] >> 62) != 0;
      if (ready) break;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((s[q] >> 62) == 0) s[q] = ld_volatile(&status[j - 4 * lane - q]);
    }
    int mine_pre = 4;  // first of my 4 entries (newest first) holding an inclusive prefix
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (mine_pre == 4 && (s[q] >> 62) == 2) mine_pre = q;
    const unsigned pre = __ballot_sync(FULL, mine_pre < 4);
    const int first = pre ? __ffs(pre) - 1 : 32;  // lane holding the nearest inclusive prefix
    uint64_t v = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t idx = j - 4 * lane - q;
      const bool take = idx >= 0 && (lane < first || (lane == first && q <= mine_pre));
      v += take ? (s[q] & LB_MASK) : 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    prefix += v;
    if (pre) break;
    j -= 128;
  }
  if (lane == 0) { st_volatile(&status[bid], LB_PRE | (prefix + agg)); }
  return prefix;
}

// --------------------------------------------------------------------------------------------
// Element prologue (compressors.py:381-411): non-finite check on the raw gradient,
// momentum (signum: b*m + (1-b)*x ; dgc: b*m + x, two roundings, no FMA), error feedback
// c = f64(work) + r (f64), c32 = f32(c).
struct Prologue {
  const float* g;
  double* r;    // null unless EF
  float* m;     // null unless momentum
  float beta, omb;
  int signum;
  __device__ __forceinline__ double load(int64_t e, float& c32, bool& bad, bool update_mom) const {
    const float x = g[e];
    bad |= !isfinite(x);
    float w = x;
    if (m) {
      const float mo = m[e];
      w = signum ? __fadd_rn(__fmul_rn(beta, mo), __fmul_rn(omb, x)) : __fadd_rn(__fmul_rn(beta, mo), x);
      if (update_mom) m[e] = w;
    }
    if (r) {
      const double c = __dadd_rn((double)w, r[e]);
      c32 = __double2float_rn(c);
      return c;
    }
    c32 = w;
    return (double)w;
  }
};

// ------------------------------------------------------------------ mbarrier + bulk copy (TMA engine, 1-D)
__device__ __forceinline__ uint32_t smem_addr(const void* ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// try_wait suspends the waiting warp (up to this many ns) instead of spinning, so waiting
// consumers do not steal issue slots from the ones computing
#ifndef MBAR_SUSPEND_NS
#define MBAR_SUSPEND_NS 20000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(MBAR_SUSPEND_NS)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// true in every thread of the last CTA of the grid to get here; the fences make all
// CTAs' earlier global writes (histogram atomics, counts) visible to it
__device__ __forceinline__ bool last_cta(uint32_t* counter) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

__device__ __forceinline__ void flag(uint32_t* err, bool bad, uint32_t bit) {
  const unsigned any = __ballot_sync(__activemask(), bad);
  if (any && (threadIdx.x & 31) == __ffs(any) - 1) atomicOr(err, bit);
}

// Sign bit position helpers: element e lives in byte e>>3 at bit 7-(e&7) (np.packbits order).
__device__ __forceinline__ uint32_t word_bit(int64_t e) { return 8u * ((e >> 3) & 3) + 7u - (e & 7); }
__device__ __forceinline__ int sign_bit(const uint8_t* bits, int64_t e) { return (bits[e >> 3] >> (7 - (e & 7))) & 1; }

// Reads code e (width w bits, MSB-first concatenation) from a packed byte stream.
__device__ __forceinline__ uint32_t read_code(const uint8_t* p, int64_t e, int w) {
  if (w == 8) return p[e];
  const int64_t bit0 = e * (int64_t)w;
  uint32_t v = 0;
  for (int b = 0; b < w; ++b) {
    const int64_t bit = bit0 + b;
    v = (v << 1) | ((p[bit >> 3] >> (7 - (bit & 7))) & 1u);
  }
  return v;
}

// Device-side header writer.
__device__ __forceinline__ void write_header(void* payload, uint32_t algo, uint32_t flags, uint64_t n, uint32_t n_idx,
                                             uint32_t n_val, uint32_t n_bits, uint32_t cap) {
  mc_payload_header* h = reinterpret_cast<mc_payload_header*>(payload);
  h->algorithm = algo; h->flags = flags; h->original_len = n; h->n_idx = n_idx; h->n_val = n_val;
  h->n_bits = n_bits; h->cap = cap;
}

// --------------------------------------------------------------------------------------------
// Entry points implemented per codec family (host side of each .cu file).
struct EncodeArgs {
  const mc_spec* spec;
  mc_layout L;
  const float* g;
  int64_t n;
  double* r;
  float* m;
  uint64_t k0, k1;
  uint8_t* payload;
  uint8_t* ws;
  int64_t ws_bytes;
  Ctx ctx;
  int64_t begin = 0;   // chunked encode: process elements [begin, begin + count) of the group
  int64_t count = -1;  // -1: the whole group
  // peer push (fused allgather over NVLink peer memory, mc_encode_push): the payload bytes
  // are also stored at push_dsts[j] (this rank's slot in rank j's gather buffer, a peer-
  // mapped device pointer; the entry equal to `payload` is skipped) and, once every CTA's
  // stores are system-visible, push_flags[j] (rank j's flag word for this rank) := epoch
  int npush = 0;
  void* const* push_dsts = nullptr;       // host array [npush] of device pointers
  uint32_t* const* push_flags = nullptr;  // host array [npush] of device pointers
  uint32_t epoch = 0;
  // graph-capturable keys (mc_encode_dk / mc_encode_decode_dk): the 128-bit Philox key is
  // read on the device from dkey[0..1] (written by mc_derive_keys) instead of (k0, k1)
  const uint64_t* dkey = nullptr;
  // NVLS multicast push (mc_encode_push_mc): multicast address of this rank's slot and flag
  void* mc_dst = nullptr;
  uint32_t* mc_flag = nullptr;
  // graph capture at N > 1: the exchange epoch read on the device (nullptr: `epoch`)
  const uint32_t* epoch_ptr = nullptr;
};

constexpr int MC_MAX_PUSH = 16;
// release-store of one flag word at system scope (readers poll with ld.acquire.sys)
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
int launch_push_copy(const uint8_t* payload, int64_t bytes, const EncodeArgs& a, cudaStream_t st,
                     const mc_layout* sparse = nullptr);

int64_t bucket_ws_bytes(const mc_spec* s, int64_t n);
int64_t sparse_ws_bytes(const mc_spec* s, int64_t n);
int64_t signglobal_ws_bytes(const mc_spec* s, int64_t n);

int encode_elementwise(const EncodeArgs& a, float* out);  // identity, fp16
// `out` (may be null / alias the gradient): also write the single-rank decoded mean in the
// same pass; returns MC_FUSED_UNSUPPORTED when the chosen path cannot (caller decodes).
constexpr int MC_FUSED_UNSUPPORTED = 1;
int encode_bucketed(const EncodeArgs& a, float* out);  // qsgd, efsignsgd, onebit, terngrad, int8
int encode_sign_global(const EncodeArgs& a);   // signsgd, signum
int encode_topk(const EncodeArgs& a, float* out);  // topk, dgc_lite (out: fused single-rank decode)
int encode_randk(const EncodeArgs& a, float* out);
int encode_threshold(const EncodeArgs& a, float* out);

int decode_mean_dense(const mc_spec* s, const mc_layout& L, const uint8_t* base, int64_t stride, int nranks,
                      float* out, const Ctx& c);
int decode_mean_sparse(const mc_spec* s, const mc_layout& L, const uint8_t* base, int64_t stride, int nranks,
                       float* out, const Ctx& c, void* ws, int64_t ws_bytes);
int64_t decode_sparse_ws_bytes(int64_t n, int nranks);

}  // namespace mc
