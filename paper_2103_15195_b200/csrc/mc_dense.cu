// mc_dense.cu — identity / fp16 encode (compressors.py:265-270) and the fused
// decode + rank-ordered mean for every dense codec (decode :450-514, aggregate :519-532).
//
// decode_mean: one thread owns 8 consecutive elements (one sign byte per rank); for
// r = 0..nranks-1 it decodes payload r and accumulates acc = fl32(acc + d_r) starting
// from +0.0f, then writes acc / f32(nranks) — the reference's float32 order exactly.
#include "mc_internal.cuh"

namespace mc {
namespace {

struct EP {
  const float* g;
  double* r;
  int64_t n;
  float* val;       // identity payload values
  __half* half;     // fp16 payload
  uint32_t* err;
  uint8_t* payload;
  mc_payload_header hdr;
  float* out;  // single-rank fused decode (may alias g)
  int write_hdr;
  int vec;  // all streams 16-byte aligned (8 for the fp16 payload): 4-wide vector path
};

template <int ALGO, bool EF, bool OUT>
__global__ void k_elementwise(EP p) {
  if (p.write_hdr && blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  bool bad = false;
  const int64_t groups = cdiv(p.n, 4);
  int64_t gstart = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!EF && p.vec) {
    // streaming fast path: U float4 groups per thread in flight (loads issued before any
    // use), so one pass keeps enough bytes outstanding per SM to run at HBM speed
    constexpr int U = 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t full_groups = p.n / 4;  // groups entirely inside the vector
    for (; gstart + (U - 1) * stride < full_groups; gstart += U * stride) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(reinterpret_cast<const float4*>(p.g) + gstart + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e0 = 4 * (gstart + u * stride);
        const float x[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
        float dec[4];
        __half h[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bad |= !isfinite(x[q]);
          if (ALGO == MC_IDENTITY) {
            dec[q] = x[q];
          } else {
            h[q] = __float2half_rn(x[q]);  // numpy astype(float16): RNE, overflow -> inf
            dec[q] = __half2float(h[q]);
          }
        }
        if (ALGO == MC_IDENTITY) {
          __stcs(reinterpret_cast<float4*>(p.val + e0), v[u]);
        } else {
          __half2 hv[2] = {__halves2half2(h[0], h[1]), __halves2half2(h[2], h[3])};
          *reinterpret_cast<uint2*>(p.half + e0) = *reinterpret_cast<uint2*>(hv);
        }
        if (OUT)  // aggregate([payload]) = (+0 + d) / 1
          __stcs(reinterpret_cast<float4*>(p.out + e0), make_float4(__fadd_rn(0.0f, dec[0]), __fadd_rn(0.0f, dec[1]),
                                                                     __fadd_rn(0.0f, dec[2]), __fadd_rn(0.0f, dec[3])));
      }
    }
  }
  for (int64_t gi = gstart; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = 4 * gi;
    const bool full = p.vec && e0 + 3 < p.n;
    float x[4];
    double rv[4] = {0.0, 0.0, 0.0, 0.0};
    if (full) {
      const float4 v = *reinterpret_cast<const float4*>(p.g + e0);
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
      if (EF) {
        const double2 a = *reinterpret_cast<const double2*>(p.r + e0), b = *reinterpret_cast<const double2*>(p.r + e0 + 2);
        rv[0] = a.x; rv[1] = a.y; rv[2] = b.x; rv[3] = b.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        x[q] = e0 + q < p.n ? p.g[e0 + q] : 0.0f;
        if (EF) rv[q] = e0 + q < p.n ? p.r[e0 + q] : 0.0;
      }
    }
    float dec[4], c32[4];
    double c[4];
    __half h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      bad |= (e0 + q < p.n) && !isfinite(x[q]);
      c[q] = EF ? __dadd_rn((double)x[q], rv[q]) : (double)x[q];
      c32[q] = EF ? __double2float_rn(c[q]) : x[q];
      if (ALGO == MC_IDENTITY) {
        dec[q] = c32[q];
      } else {
        h[q] = __float2half_rn(c32[q]);  // numpy astype(float16): RNE, overflow -> inf
        dec[q] = __half2float(h[q]);
      }
    }
    if (full) {
      if (ALGO == MC_IDENTITY) *reinterpret_cast<float4*>(p.val + e0) = make_float4(c32[0], c32[1], c32[2], c32[3]);
      else {
        __half2 hv[2] = {__halves2half2(h[0], h[1]), __halves2half2(h[2], h[3])};
        *reinterpret_cast<uint2*>(p.half + e0) = *reinterpret_cast<uint2*>(hv);
      }
      if (EF) {
        *reinterpret_cast<double2*>(p.r + e0) = make_double2(__dsub_rn(c[0], (double)dec[0]), __dsub_rn(c[1], (double)dec[1]));
        *reinterpret_cast<double2*>(p.r + e0 + 2) = make_double2(__dsub_rn(c[2], (double)dec[2]), __dsub_rn(c[3], (double)dec[3]));
      }
      if (OUT)  // aggregate([payload]) = (+0 + d) / 1
        *reinterpret_cast<float4*>(p.out + e0) = make_float4(__fadd_rn(0.0f, dec[0]), __fadd_rn(0.0f, dec[1]),
                                                             __fadd_rn(0.0f, dec[2]), __fadd_rn(0.0f, dec[3]));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t e = e0 + q;
        if (e >= p.n) break;
        if (ALGO == MC_IDENTITY) p.val[e] = c32[q];
        else p.half[e] = h[q];
        if (EF) p.r[e] = __dsub_rn(c[q], (double)dec[q]);
        if (OUT) p.out[e] = __fadd_rn(0.0f, dec[q]);
      }
    }
  }
  flag(p.err, bad, MC_ERR_NONFINITE);
}

// ------------------------------------------------------------------ dense decode
struct DP {
  const uint8_t* base;
  int64_t stride;
  int nranks;
  int64_t n, B;
  int64_t off_val, off_bits, off_codes;
  int width;
  float top;
  float inv_unused;
  float* out;
  uint32_t* err;
  uint32_t algo;
  uint32_t n_val, n_bits;
};

// Decode 8 consecutive elements e0 .. e0+7 (e0 % 8 == 0) of one payload.  SAMEB: the 8
// elements share one bucket (bucket_size % 8 == 0) — one scale load, one sign byte.
template <int ALGO, bool SAMEB>
__device__ __forceinline__ void dec8(const DP& p, const uint8_t* pl, uint32_t e0, int cnt, float (&d)[8]) {
  const float* val = reinterpret_cast<const float*>(pl + p.off_val);
  const uint8_t* bits = pl + p.off_bits;
  if (ALGO == MC_IDENTITY) {
    if (cnt == 8) {
      const float4 a = reinterpret_cast<const float4*>(val + e0)[0], b = reinterpret_cast<const float4*>(val + e0)[1];
      d[0] = a.x; d[1] = a.y; d[2] = a.z; d[3] = a.w; d[4] = b.x; d[5] = b.y; d[6] = b.z; d[7] = b.w;
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = q < cnt ? val[e0 + q] : 0.0f;
    }
    return;
  }
  if (ALGO == MC_FP16) {
    const __half* h = reinterpret_cast<const __half*>(bits) + e0;
    if (cnt == 8) {
      const uint4 v = *reinterpret_cast<const uint4*>(h);
      const __half2* h2 = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __half22float2(h2[q]);
        d[2 * q] = f.x;
        d[2 * q + 1] = f.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = q < cnt ? __half2float(h[q]) : 0.0f;
    }
    return;
  }
  if (ALGO == MC_TERNGRAD) {
    const uint32_t w = bits[e0 >> 2] << 8 | (cnt > 4 ? bits[(e0 >> 2) + 1] : 0u);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float s = val[SAMEB ? e0 / (uint32_t)p.B : (e0 + q) / (uint32_t)p.B];
      const uint32_t code = (w >> (14 - 2 * q)) & 3u;
      d[q] = __fmul_rn(__fsub_rn((float)code, 1.0f), s);  // (code - 1) * s   (:501-504)
    }
    return;
  }
  if (ALGO == MC_INT8) {
    uint64_t w = 0;
    if (cnt == 8) w = *reinterpret_cast<const uint64_t*>(bits + e0);
    else
      for (int q = 0; q < cnt; ++q) w |= (uint64_t)bits[e0 + q] << (8 * q);
    const float step0 = __fdiv_rn(val[e0 / (uint32_t)p.B], 127.0f);  // s / 127 of the group's bucket
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float step = SAMEB ? step0 : __fdiv_rn(val[(e0 + q) / (uint32_t)p.B], 127.0f);
      d[q] = __fmul_rn((float)(int8_t)(uint8_t)(w >> (8 * q)), step);  // q * (s / 127)  (:513)
    }
    return;
  }
  // sign family: one byte carries the 8 signs, MSB = e0
  const uint32_t sb = bits[e0 >> 3];
  uint64_t codes8 = 0;
  if (ALGO == MC_QSGD && p.width == 8) {
    const uint8_t* cp = pl + p.off_codes;
    if (cnt == 8) codes8 = *reinterpret_cast<const uint64_t*>(cp + e0);
    else
      for (int q = 0; q < cnt; ++q) codes8 |= (uint64_t)cp[e0 + q] << (8 * q);
  }
  const uint32_t b0 = (ALGO == MC_SIGNSGD || ALGO == MC_SIGNUM) ? 0u : e0 / (uint32_t)p.B;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t b = SAMEB ? b0 : (ALGO == MC_SIGNSGD || ALGO == MC_SIGNUM) ? 0u : (e0 + q) / (uint32_t)p.B;
    const float sgn = ((sb >> (7 - q)) & 1u) ? 1.0f : -1.0f;
    if (ALGO == MC_SIGNSGD || ALGO == MC_SIGNUM) d[q] = __fmul_rn(sgn, val[0]);
    else if (ALGO == MC_EFSIGNSGD) d[q] = __fmul_rn(sgn, val[b]);
    else if (ALGO == MC_ONEBIT) d[q] = ((sb >> (7 - q)) & 1u) ? val[2 * b + 1] : val[2 * b];
    else {  // MC_QSGD: (sign * s) * (code / (L-1))   (:470)
      const uint32_t code = p.width == 8 ? (uint32_t)((codes8 >> (8 * q)) & 0xffu)
                                         : (q < cnt ? read_code(pl + p.off_codes, e0 + q, p.width) : 0u);
      d[q] = __fmul_rn(__fmul_rn(sgn, val[b]), __fdiv_rn((float)code, p.top));
    }
  }
}

// acc / f32(nranks): for a power-of-two rank count the product with the exact reciprocal
// is the same correctly rounded value as the IEEE quotient (both round the same real).
__device__ __forceinline__ float rank_mean(float acc, float fn, float inv, bool pow2) {
  return pow2 ? __fmul_rn(acc, inv) : __fdiv_rn(acc, fn);
}

// Sign-bit codecs (efsignsgd, onebit, signsgd/signum, 8-bit qsgd): one thread per 32-element
// sign word, bucket_size % 32 == 0 so the word lies in one bucket; per rank one u32 of
// signs + the bucket scale(s) (+ 32 code bytes), per element select/multiply + add.
// qsgd's code / (L-1) comes from a 256-entry table of the exact IEEE quotients.
// symmetric +-scale codecs: 4 CTAs per SM (64 registers) — the N-rank accumulation is
// issue-bound and occupancy hides its dependent adds (efsignsgd N=8: 43 -> 39 us); onebit
// and qsgd keep more registers (two scales per bucket / the code table)
template <int ALGO>
__global__ void __launch_bounds__(256, (ALGO == MC_QSGD || ALGO == MC_ONEBIT) ? 1 : 4) k_decode_sign32(DP p) {
  __shared__ float tbl[256];
  __shared__ __align__(16) float s_out[8][32 * 36];
  if (ALGO == MC_QSGD) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tbl[i] = __fdiv_rn((float)i, p.top);
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x < p.nranks) {
    const mc_payload_header* h = reinterpret_cast<const mc_payload_header*>(p.base + p.stride * threadIdx.x);
    if (h->algorithm != p.algo || h->original_len != (uint64_t)p.n || h->n_val != p.n_val || h->n_bits != p.n_bits)
      atomicOr(p.err, MC_ERR_HEADER);
  }
  const float fn = (float)p.nranks;
  const bool pow2 = (p.nranks & (p.nranks - 1)) == 0;
  const float inv = __fdiv_rn(1.0f, fn);
  const uint32_t words = (uint32_t)cdiv(p.n, 32);
  const bool vout = ((uintptr_t)p.out % 16) == 0;
  const int lane = threadIdx.x & 31;
  float* so = s_out[threadIdx.x >> 5];
  // warp-uniform loop: lane l owns word wb + l (32 consecutive words = 1024 elements)
  for (uint32_t wb = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wb < words; wb += gridDim.x * blockDim.x) {
    const uint32_t w = wb + lane;
    const bool live = w < words;
    const uint32_t e0 = 32 * w;
    const int cnt = live ? (int)imin(32, p.n - (int64_t)e0) : 0;
    const uint32_t b = (ALGO == MC_SIGNSGD || ALGO == MC_SIGNUM) ? 0u : e0 / (uint32_t)p.B;
    float acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = 0.0f;
    // ranks in chunks of RC: all loads of a chunk are issued before any use (ILP across
    // ranks); accumulation stays in rank order 0..n-1 (compressors.py:529-531)
    constexpr int RC = (ALGO == MC_QSGD) ? 4 : 8;
    for (int r0 = 0; r0 < p.nranks; r0 += RC) {
      uint32_t sw[RC];
      float hi[RC], lo[RC];
      uint32_t cw[ALGO == MC_QSGD ? RC : 1][8];
#pragma unroll
      for (int rr = 0; rr < RC; ++rr) {
        sw[rr] = 0;
        hi[rr] = lo[rr] = 0.0f;
        if (r0 + rr >= p.nranks || !live) continue;
        const uint8_t* pl = p.base + p.stride * (r0 + rr);
        const float* val = reinterpret_cast<const float*>(pl + p.off_val);
        sw[rr] = reinterpret_cast<const uint32_t*>(pl + p.off_bits)[w];
        if (ALGO == MC_ONEBIT) { lo[rr] = val[2 * b]; hi[rr] = val[2 * b + 1]; }
        else { hi[rr] = val[b]; }
        if (ALGO == MC_QSGD) {
          const uint8_t* cp = pl + p.off_codes + e0;
          if (cnt == 32) {
            const uint4 c0 = reinterpret_cast<const uint4*>(cp)[0], c1 = reinterpret_cast<const uint4*>(cp)[1];
            cw[ALGO == MC_QSGD ? rr : 0][0] = c0.x; cw[ALGO == MC_QSGD ? rr : 0][1] = c0.y;
            cw[ALGO == MC_QSGD ? rr : 0][2] = c0.z; cw[ALGO == MC_QSGD ? rr : 0][3] = c0.w;
            cw[ALGO == MC_QSGD ? rr : 0][4] = c1.x; cw[ALGO == MC_QSGD ? rr : 0][5] = c1.y;
            cw[ALGO == MC_QSGD ? rr : 0][6] = c1.z; cw[ALGO == MC_QSGD ? rr : 0][7] = c1.w;
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint32_t v = 0;
              for (int t = 0; t < 4; ++t)
                if (4 * j + t < cnt) v |= (uint32_t)cp[4 * j + t] << (8 * t);
              cw[ALGO == MC_QSGD ? rr : 0][j] = v;
            }
          }
        }
      }
#pragma unroll
      for (int rr = 0; rr < RC; ++rr) {
        if (r0 + rr >= p.nranks) break;
        if (ALGO != MC_ONEBIT) lo[rr] = __fmul_rn(-1.0f, hi[rr]);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const bool bit = (sw[rr] >> (8 * (q >> 3) + 7 - (q & 7))) & 1u;  // np.packbits order
          float d = bit ? hi[rr] : lo[rr];
          if (ALGO == MC_QSGD)  // (sgn * s) * (code / (L-1))
            d = __fmul_rn(d, tbl[(cw[ALGO == MC_QSGD ? rr : 0][q >> 2] >> (8 * (q & 3))) & 0xffu]);
          acc[q] = __fadd_rn(acc[q], d);
        }
      }
    }
    if (__all_sync(FULL, cnt == 32) && vout) {
      // transpose through shared memory (rows of 36 floats: conflict-free float4 in and
      // out) so each warp-wide store is one contiguous 512-byte row of the output
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(so + 36 * lane + 4 * j) =
            make_float4(rank_mean(acc[4 * j], fn, inv, pow2), rank_mean(acc[4 * j + 1], fn, inv, pow2),
                        rank_mean(acc[4 * j + 2], fn, inv, pow2), rank_mean(acc[4 * j + 3], fn, inv, pow2));
      __syncwarp();
      float* ob = p.out + (int64_t)32 * wb;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int idx = 128 * j + 4 * lane;
        reinterpret_cast<float4*>(ob)[32 * j + lane] = *reinterpret_cast<const float4*>(so + 36 * (idx >> 5) + (idx & 31));
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q < cnt) p.out[e0 + q] = rank_mean(acc[q], fn, inv, pow2);
    }
  }
}

// Sign codecs over 3..8 ranks by table.  Every rank's decoded value of an element is one of
// two per-bucket constants (+-s, or onebit's two means), so the rank-ordered f32 sum
// 0 + d_0 + ... + d_{N-1} (compressors.py:529-531) and its mean depend only on the element's
// N sign bits: a warp first builds, for each bucket its 1024 elements touch, the table
// T[pattern] of all 2^N exact rank-ordered means (the first min(N, 4) ranks' partial sums
// once per lane, then the remaining ranks per entry — the same additions in the same
// order as the per-element loop), then turns its 32 words x N ranks of sign bits into one
// N-bit pattern per element with 8x8 bit transposes and reads the mean from the table.
// Per element: a few transpose ops + a table read instead of N selects + N adds
// (ResNet-50 set, efsignsgd: N=4 32.4 -> 24.6 us, N=8 39.2 -> 34.9 us).
constexpr int TAB_FLOATS = 512;  // per-warp table budget (buckets per warp x 2^N)
constexpr int TAB_STAGE_FLOATS = 32 * 36;  // output rows staged for 512-byte stores (direct
                                           // per-lane float4 stores measured 40% slower)
template <int ALGO, int N>
__global__ void __launch_bounds__(256) k_decode_sign_tab(DP p) {
  constexpr bool WHOLE = (ALGO == MC_SIGNSGD || ALGO == MC_SIGNUM);  // one scale per rank
  constexpr int L1 = N < 4 ? N : 4, H = N - L1;
  extern __shared__ __align__(16) float dsm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* tab = dsm + warp * (TAB_FLOATS + TAB_STAGE_FLOATS);
  float* so = tab + TAB_FLOATS;
  if (blockIdx.x == 0 && threadIdx.x < N) {
    const mc_payload_header* h = reinterpret_cast<const mc_payload_header*>(p.base + p.stride * threadIdx.x);
    if (h->algorithm != p.algo || h->original_len != (uint64_t)p.n || h->n_val != p.n_val || h->n_bits != p.n_bits)
      atomicOr(p.err, MC_ERR_HEADER);
  }
  const float fn = (float)N;
  constexpr bool POW2 = (N & (N - 1)) == 0;
  const float inv = __fdiv_rn(1.0f, fn);
  const uint32_t words = (uint32_t)cdiv(p.n, 32);
  const int64_t nb = WHOLE ? 1 : cdiv(p.n, p.B);
  const bool vout = ((uintptr_t)p.out % 16) == 0;
  for (uint32_t wb = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); wb < words; wb += gridDim.x * blockDim.x) {
    // sign words first: their loads are in flight while the tables are built
    const uint32_t w = wb + lane;
    const bool live = w < words;
    const int cnt = live ? (int)imin(32, p.n - (int64_t)32 * w) : 0;
    uint32_t sw[8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
      sw[r] = (r < N && live) ? reinterpret_cast<const uint32_t*>(p.base + p.stride * r + p.off_bits)[w] : 0u;
    // ---- tables of the buckets under words wb .. wb+31
    const int64_t b_first = WHOLE ? 0 : (int64_t)32 * wb / p.B;
    const int64_t b_last = WHOLE ? 0 : imin(nb - 1, ((int64_t)32 * (wb + 31) + 31) / p.B);
    const int nbw = (int)(b_last - b_first + 1);
    for (int pi = lane; pi < (nbw << H); pi += 32) {
      const int j = pi >> H, h = pi & ((1 << H) - 1);
      const int64_t b = b_first + j;
      float hi[N], lo[N];
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const float* val = reinterpret_cast<const float*>(p.base + p.stride * r + p.off_val);
        if (ALGO == MC_ONEBIT) { lo[r] = val[2 * b]; hi[r] = val[2 * b + 1]; }
        else { hi[r] = val[b]; lo[r] = __fmul_rn(-1.0f, hi[r]); }
      }
      float t[1 << L1];  // partial sums over ranks 0..L1-1 for every low pattern u
      t[0] = 0.0f;
#pragma unroll
      for (int r = 0; r < L1; ++r)
#pragma unroll
        for (int u = (1 << r) - 1; u >= 0; --u) {  // in place: t[u | 1<<r] from t[u] first
          t[u | (1 << r)] = __fadd_rn(t[u], hi[r]);
          t[u] = __fadd_rn(t[u], lo[r]);
        }
#pragma unroll
      for (int u = 0; u < (1 << L1); ++u) {
        float acc = t[u];
#pragma unroll
        for (int r = L1; r < N; ++r) acc = __fadd_rn(acc, ((h >> (r - L1)) & 1) ? hi[r] : lo[r]);
        tab[(j << N) | (h << L1) | u] = rank_mean(acc, fn, inv, POW2);
      }
    }
    __syncwarp();
    // ---- per element: N sign bits -> pattern -> mean
    const float* tb = tab + ((WHOLE ? 0 : (int)((int64_t)32 * w / p.B - b_first)) << N);
    float v[32];
#pragma unroll
    for (int jb = 0; jb < 4; ++jb) {  // byte jb of the word: elements 8 jb .. 8 jb + 7
      uint32_t xl = 0, xh = 0;  // byte r of x = byte jb of rank r's word
#pragma unroll
      for (int r = 0; r < 4; ++r) xl |= ((sw[r] >> (8 * jb)) & 0xffu) << (8 * r);
#pragma unroll
      for (int r = 0; r < 4; ++r) xh |= ((sw[r + 4] >> (8 * jb)) & 0xffu) << (8 * r);
      uint64_t x = ((uint64_t)xh << 32) | xl, t;  // 8x8 bit transpose: bit 8r+c <-> bit 8c+r
      t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull; x ^= t ^ (t << 7);
      t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull; x ^= t ^ (t << 14);
      t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull; x ^= t ^ (t << 28);
#pragma unroll
      for (int c = 0; c < 8; ++c)  // byte c of x: the pattern of element 8 jb + 7 - c (np.packbits)
        v[8 * jb + 7 - c] = tb[(uint32_t)(x >> (8 * c)) & ((1u << N) - 1u)];
    }
    if (__all_sync(FULL, cnt == 32) && vout) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(so + 36 * lane + 4 * j) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      __syncwarp();
      float* ob = p.out + (int64_t)32 * wb;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int idx = 128 * j + 4 * lane;
        reinterpret_cast<float4*>(ob)[32 * j + lane] = *reinterpret_cast<const float4*>(so + 36 * (idx >> 5) + (idx & 31));
      }
    } else {
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q < cnt) p.out[(int64_t)32 * w + q] = v[q];
    }
    __syncwarp();  // the table and staging rows are rewritten by the next iteration
  }
}

template <int ALGO>
int launch_sign_tab(const DP& p, cudaStream_t st) {
  constexpr int smem = 8 * (TAB_FLOATS + TAB_STAGE_FLOATS) * 4;
  static std::atomic<uint64_t> configured[6];
  const unsigned grid = (unsigned)imax(1, imin(cdiv(cdiv(p.n, 32), 256), (int64_t)sm_count() * 4));
#define MC_TAB(NR)                                                                               \
  case NR:                                                                                       \
    if (smem_optin(configured[NR - 3], k_decode_sign_tab<ALGO, NR>, smem) != cudaSuccess) {      \
      set_error("cudaFuncSetAttribute(%d bytes smem) failed", smem);                            \
      return MC_ECUDA;                                                                           \
    }                                                                                            \
    note_launch();                                                                               \
    k_decode_sign_tab<ALGO, NR><<<grid, 256, smem, st>>>(p);                                     \
    break;
  switch (p.nranks) {
    MC_TAB(3) MC_TAB(4) MC_TAB(5) MC_TAB(6) MC_TAB(7) MC_TAB(8)
    default: return MC_EINVAL;
  }
#undef MC_TAB
  MC_LAUNCH_CHECK();
  return MC_OK;
}

// One payload of a whole-group scale (signsgd / signum, world size 1): out = bit ? s : -s
// (compressors.py:476-481, then aggregate's 0 + d / f32(1)).  A warp expands 1024
// elements: lane l loads sign word l, and every store is one contiguous 512-byte row built
// from the word of lane 4j + l/8 (a shuffle) — pure streaming writes.
__global__ void __launch_bounds__(256) k_decode_sign_one(DP p) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const mc_payload_header* h = reinterpret_cast<const mc_payload_header*>(p.base);
    if (h->algorithm != p.algo || h->original_len != (uint64_t)p.n || h->n_val != p.n_val || h->n_bits != p.n_bits)
      atomicOr(p.err, MC_ERR_HEADER);
  }
  const float s = __fadd_rn(0.0f, reinterpret_cast<const float*>(p.base + p.off_val)[0]);
  const float ns = __fadd_rn(0.0f, __fmul_rn(-1.0f, reinterpret_cast<const float*>(p.base + p.off_val)[0]));
  const uint32_t* words = reinterpret_cast<const uint32_t*>(p.base + p.off_bits);
  const int lane = threadIdx.x & 31;
  const int64_t nwords = cdiv(p.n, 32);
  const bool vout = ((uintptr_t)p.out % 16) == 0;
  const int64_t wstride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t wb = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); wb < nwords; wb += wstride) {
    const uint32_t mine = wb + lane < nwords ? words[wb + lane] : 0u;
    const int64_t e_base = 32 * wb;
    const bool full = vout && e_base + 1024 <= p.n;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t wv = __shfl_sync(FULL, mine, 4 * j + (lane >> 3));
      const int sh = 8 * ((lane >> 1) & 3) + ((lane & 1) ? 0 : 4);  // nibble of elements 4l..4l+3
      const uint32_t nib = (wv >> sh) & 0xfu;
      const float4 v = make_float4((nib & 8) ? s : ns, (nib & 4) ? s : ns, (nib & 2) ? s : ns, (nib & 1) ? s : ns);
      const int64_t e0 = e_base + 128 * j + 4 * lane;
      if (full) {
        __stcs(reinterpret_cast<float4*>(p.out + e0), v);
      } else {
        const float vv[4] = {v.x, v.y, v.z, v.w};
        for (int q = 0; q < 4; ++q)
          if (e0 + q < p.n) p.out[e0 + q] = vv[q];
      }
    }
  }
}

// Byte codecs over N ranks (identity / fp16 / int8 / terngrad, bucket_size % 8 == 0): 8 elements per
// thread, ranks in chunks of RC whose loads are all issued before any is used (the per-rank
// loop of k_decode_dense leaves one rank's load in flight per thread and is latency-bound).
// ResNet-50 set: int8 N=4/8 77 -> 57 / 132 -> 87 us, fp16 60 -> 55 / 100 -> 80 us (its HBM
// floor: 78 us), identity N=8 138 us (floor 141).  Accumulation stays in rank order
// (compressors.py:529-531).
template <int ALGO>
__global__ void __launch_bounds__(256) k_decode_bytes(DP p) {
  constexpr int RC = ALGO == MC_IDENTITY ? 4 : 8;
  __shared__ float tbl[ALGO == MC_QSGD ? 256 : 1];
  if (ALGO == MC_QSGD) {  // exact IEEE quotients code / (L-1)
    tbl[threadIdx.x] = __fdiv_rn((float)threadIdx.x, p.top);
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x < p.nranks) {
    const mc_payload_header* h = reinterpret_cast<const mc_payload_header*>(p.base + p.stride * threadIdx.x);
    if (h->algorithm != p.algo || h->original_len != (uint64_t)p.n || h->n_val != p.n_val || h->n_bits != p.n_bits)
      atomicOr(p.err, MC_ERR_HEADER);
  }
  const float fn = (float)p.nranks;
  const bool pow2 = (p.nranks & (p.nranks - 1)) == 0;
  const float inv = __fdiv_rn(1.0f, fn);
  const uint32_t groups = (uint32_t)cdiv(p.n, 8);
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += gridDim.x * blockDim.x) {
    const uint32_t e0 = gi * 8;
    const int cnt = (int)imin(8, p.n - (int64_t)e0);
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
    if (cnt < 8) {  // the group's ragged end
      for (int r = 0; r < p.nranks; ++r) {
        float d[8];
        dec8<ALGO, true>(p, p.base + p.stride * r, e0, cnt, d);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], d[q]);
      }
    } else {
      const uint32_t b = e0 / (uint32_t)p.B;
      for (int r0 = 0; r0 < p.nranks; r0 += RC) {
        uint4 raw[RC][ALGO == MC_IDENTITY ? 2 : 1];
        float sc[RC];
        const int nr = p.nranks - r0 < RC ? p.nranks - r0 : RC;
#pragma unroll
        for (int rr = 0; rr < RC; ++rr) {  // every load of the chunk first
          if (rr >= nr) continue;
          const uint8_t* pl = p.base + p.stride * (r0 + rr);
          if (ALGO == MC_IDENTITY) {
            const uint4* v = reinterpret_cast<const uint4*>(pl + p.off_val) + 2 * (size_t)gi;
            raw[rr][0] = v[0];
            raw[rr][ALGO == MC_IDENTITY ? 1 : 0] = v[1];
          } else if (ALGO == MC_FP16) {
            raw[rr][0] = reinterpret_cast<const uint4*>(pl + p.off_bits)[gi];
          } else if (ALGO == MC_QSGD) {  // 8 code bytes, the sign byte (MSB = first) + the scale
            const uint2 c = reinterpret_cast<const uint2*>(pl + p.off_codes)[gi];
            raw[rr][0] = make_uint4(c.x, c.y, (uint32_t)(pl + p.off_bits)[gi], 0u);
            sc[rr] = reinterpret_cast<const float*>(pl + p.off_val)[b];
          } else if (ALGO == MC_TERNGRAD) {  // 8 two-bit codes (MSB-first) + the bucket scale
            const uint16_t c = reinterpret_cast<const uint16_t*>(pl + p.off_bits)[gi];
            raw[rr][0] = make_uint4((uint32_t)c, 0u, 0u, 0u);
            sc[rr] = reinterpret_cast<const float*>(pl + p.off_val)[b];
          } else {  // int8: 8 code bytes + the bucket scale
            const uint2 c = reinterpret_cast<const uint2*>(pl + p.off_bits)[gi];
            raw[rr][0] = make_uint4(c.x, c.y, 0u, 0u);
            sc[rr] = reinterpret_cast<const float*>(pl + p.off_val)[b];
          }
        }
#pragma unroll
        for (int rr = 0; rr < RC; ++rr) {
          if (rr >= nr) continue;
          float d[8];
          if (ALGO == MC_IDENTITY) {
            const uint4 a = raw[rr][0], c = raw[rr][ALGO == MC_IDENTITY ? 1 : 0];
            d[0] = __uint_as_float(a.x); d[1] = __uint_as_float(a.y); d[2] = __uint_as_float(a.z);
            d[3] = __uint_as_float(a.w); d[4] = __uint_as_float(c.x); d[5] = __uint_as_float(c.y);
            d[6] = __uint_as_float(c.z); d[7] = __uint_as_float(c.w);
          } else if (ALGO == MC_FP16) {
            const __half2* h2 = reinterpret_cast<const __half2*>(&raw[rr][0]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 f = __half22float2(h2[q]);
              d[2 * q] = f.x;
              d[2 * q + 1] = f.y;
            }
          } else if (ALGO == MC_QSGD) {  // (sign * s) * (code / (L-1))  (:470)
            const float s = sc[rr], ns = __fmul_rn(-1.0f, s);
            const uint32_t lo = raw[rr][0].x, hi = raw[rr][0].y, sb = raw[rr][0].z;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t code = ((q < 4 ? lo : hi) >> (8 * (q & 3))) & 0xffu;
              d[q] = __fmul_rn(((sb >> (7 - q)) & 1u) ? s : ns, tbl[code]);
            }
          } else if (ALGO == MC_TERNGRAD) {  // (code - 1) * s  (:501-504)
            const uint32_t w = raw[rr][0].x;  // byte 0 = elements 0..3, byte 1 = elements 4..7
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const uint32_t code = (w >> (8 * (q >> 2) + 6 - 2 * (q & 3))) & 3u;
              d[q] = __fmul_rn(__fsub_rn((float)code, 1.0f), sc[rr]);
            }
          } else {
            const float step = __fdiv_rn(sc[rr], 127.0f);  // s / 127  (:513)
            const uint64_t w = (uint64_t)raw[rr][0].x | ((uint64_t)raw[rr][0].y << 32);
#pragma unroll
            for (int q = 0; q < 8; ++q) d[q] = __fmul_rn((float)(int8_t)(uint8_t)(w >> (8 * q)), step);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], d[q]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = rank_mean(acc[q], fn, inv, pow2);
    if (cnt == 8) {
      reinterpret_cast<float4*>(p.out + e0)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      reinterpret_cast<float4*>(p.out + e0)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < cnt) p.out[e0 + q] = acc[q];
    }
  }
}

template <int ALGO, bool SAMEB>
__global__ void __launch_bounds__(256) k_decode_dense(DP p) {
  if (blockIdx.x == 0 && threadIdx.x < p.nranks) {
    const mc_payload_header* h = reinterpret_cast<const mc_payload_header*>(p.base + p.stride * threadIdx.x);
    if (h->algorithm != p.algo || h->original_len != (uint64_t)p.n || h->n_val != p.n_val || h->n_bits != p.n_bits)
      atomicOr(p.err, MC_ERR_HEADER);
  }
  const float fn = (float)p.nranks;
  const bool pow2 = (p.nranks & (p.nranks - 1)) == 0;
  const float inv = __fdiv_rn(1.0f, fn);
  const uint32_t groups = (uint32_t)cdiv(p.n, 8);
  const bool vout = ((uintptr_t)p.out % 16) == 0;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += gridDim.x * blockDim.x) {
    const uint32_t e0 = gi * 8;
    const int cnt = (int)imin(8, p.n - (int64_t)e0);
    float acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
#pragma unroll 4
    for (int r = 0; r < p.nranks; ++r) {  // rank order 0..n-1, fp32 (compressors.py:529-531)
      float d[8];
      dec8<ALGO, SAMEB>(p, p.base + p.stride * r, e0, cnt, d);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = __fadd_rn(acc[q], d[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = rank_mean(acc[q], fn, inv, pow2);
    if (cnt == 8 && vout) {
      reinterpret_cast<float4*>(p.out + e0)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      reinterpret_cast<float4*>(p.out + e0)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < cnt) p.out[e0 + q] = acc[q];
    }
  }
}

}  // namespace

int encode_elementwise(const EncodeArgs& a, float* out) {
  const mc_spec* s = a.spec;
  const int64_t begin = a.begin, count = a.count < 0 ? a.n - a.begin : a.count;
  EP p{};
  p.g = a.g + begin;
  p.r = s->error_feedback ? a.r + begin : nullptr;
  p.n = count;
  p.val = reinterpret_cast<float*>(a.payload + a.L.off_val) + begin;
  p.half = reinterpret_cast<__half*>(a.payload + a.L.off_bits) + begin;
  p.err = a.ctx.err;
  p.payload = a.payload;
  p.out = out ? out + begin : nullptr;
  p.write_hdr = begin == 0;
  p.vec = ((uintptr_t)p.g % 16 == 0) && (!p.r || (uintptr_t)p.r % 16 == 0) && ((uintptr_t)p.val % 16 == 0) &&
          ((uintptr_t)p.half % 8 == 0) && (!p.out || (uintptr_t)p.out % 16 == 0);
  p.hdr.algorithm = (uint32_t)s->algorithm;
  p.hdr.original_len = (uint64_t)a.n;
  p.hdr.n_val = (uint32_t)a.L.n_val;
  p.hdr.n_bits = (uint32_t)a.L.n_bits;
  const unsigned grid = (unsigned)imax(1, imin(cdiv(count, 1024), (int64_t)sm_count() * 16));
  cudaStream_t st = a.ctx.stream;
  note_launch();
#define MC_EW(A, EF, OUT) k_elementwise<A, EF, OUT><<<grid, 256, 0, st>>>(p)
  if (s->algorithm == MC_IDENTITY) {
    if (p.r) { if (out) MC_EW(MC_IDENTITY, true, true); else MC_EW(MC_IDENTITY, true, false); }
    else { if (out) MC_EW(MC_IDENTITY, false, true); else MC_EW(MC_IDENTITY, false, false); }
  } else {
    if (p.r) { if (out) MC_EW(MC_FP16, true, true); else MC_EW(MC_FP16, true, false); }
    else { if (out) MC_EW(MC_FP16, false, true); else MC_EW(MC_FP16, false, false); }
  }
#undef MC_EW
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int decode_mean_dense(const mc_spec* s, const mc_layout& L, const uint8_t* base, int64_t stride, int nranks,
                      float* out, const Ctx& c) {
  DP p{};
  p.base = base;
  p.stride = stride;
  p.nranks = nranks;
  p.n = L.n;
  p.B = s->bucket_size;
  p.off_val = L.off_val;
  p.off_bits = L.off_bits;
  p.off_codes = L.off_codes;
  p.width = level_bits(s->levels);
  p.top = (float)(s->levels - 1);
  p.out = out;
  p.err = c.err;
  p.algo = (uint32_t)s->algorithm;
  p.n_val = (uint32_t)L.n_val;
  p.n_bits = (uint32_t)(L.n_bits + L.n_codes);
  const int64_t groups = cdiv(L.n, 8);
  const unsigned grid = (unsigned)imax(1, imin(cdiv(groups, 256), (int64_t)sm_count() * 16));
  cudaStream_t st = c.stream;
  const bool sameb = p.B % 8 == 0;
  const int a = s->algorithm;
  const bool sign32 = (a == MC_SIGNSGD || a == MC_SIGNUM) ||
                      ((a == MC_EFSIGNSGD || a == MC_ONEBIT || (a == MC_QSGD && p.width == 8)) && p.B % 32 == 0);
  if ((a == MC_SIGNSGD || a == MC_SIGNUM) && nranks == 1) {
    const unsigned g1 = (unsigned)imax(1, imin(cdiv(cdiv(L.n, 32), 256), (int64_t)sm_count() * 8));
    note_launch();
    k_decode_sign_one<<<g1, 256, 0, st>>>(p);
    MC_LAUNCH_CHECK();
    return MC_OK;
  }
  // table decode: 3..8 ranks, the per-warp tables of the buckets under 1024 elements fit
  const bool tab_ok = nranks >= 3 && nranks <= 8 && (a == MC_SIGNSGD || a == MC_SIGNUM ||
      ((a == MC_EFSIGNSGD || a == MC_ONEBIT) && p.B % 32 == 0 &&
       (1024 % p.B == 0 ? 1024 / p.B : 1023 / p.B + 2) << nranks <= TAB_FLOATS));
  if (tab_ok) {
    switch (a) {
      case MC_SIGNSGD: return launch_sign_tab<MC_SIGNSGD>(p, st);
      case MC_SIGNUM: return launch_sign_tab<MC_SIGNUM>(p, st);
      case MC_EFSIGNSGD: return launch_sign_tab<MC_EFSIGNSGD>(p, st);
      default: return launch_sign_tab<MC_ONEBIT>(p, st);
    }
  }
  // byte codecs with aligned sections: the chunk-prefetching kernel (alignment of every
  // rank's sections follows from the 16-byte aligned layout and a 16-byte stride)
  const bool aligned = stride % 16 == 0 && (uintptr_t)base % 16 == 0 && (uintptr_t)out % 16 == 0;
  // (fp16 / identity / terngrad at 2-3 ranks stay on k_decode_dense and 8-bit qsgd below 8
  // ranks on k_decode_sign32: more resident warps, measured faster; qsgd at 8 ranks
  // 122 -> 113 us on ResNet-50)
  if (aligned && sameb && ((a == MC_INT8 && nranks > 1) || (a == MC_QSGD && p.width == 8 && nranks >= 8) ||
                           ((a == MC_IDENTITY || a == MC_FP16 || a == MC_TERNGRAD) && nranks >= 4))) {
    note_launch();
    if (a == MC_QSGD) k_decode_bytes<MC_QSGD><<<grid, 256, 0, st>>>(p);
    else if (a == MC_IDENTITY) k_decode_bytes<MC_IDENTITY><<<grid, 256, 0, st>>>(p);
    else if (a == MC_FP16) k_decode_bytes<MC_FP16><<<grid, 256, 0, st>>>(p);
    else if (a == MC_TERNGRAD) k_decode_bytes<MC_TERNGRAD><<<grid, 256, 0, st>>>(p);
    else k_decode_bytes<MC_INT8><<<grid, 256, 0, st>>>(p);
    MC_LAUNCH_CHECK();
    return MC_OK;
  }
  if (sign32) {
    const unsigned g32 = (unsigned)imax(1, imin(cdiv(cdiv(L.n, 32), 256), (int64_t)sm_count() * 8));
    note_launch();
    switch (a) {
      case MC_SIGNSGD: k_decode_sign32<MC_SIGNSGD><<<g32, 256, 0, st>>>(p); break;
      case MC_SIGNUM: k_decode_sign32<MC_SIGNUM><<<g32, 256, 0, st>>>(p); break;
      case MC_EFSIGNSGD: k_decode_sign32<MC_EFSIGNSGD><<<g32, 256, 0, st>>>(p); break;
      case MC_ONEBIT: k_decode_sign32<MC_ONEBIT><<<g32, 256, 0, st>>>(p); break;
      default: k_decode_sign32<MC_QSGD><<<g32, 256, 0, st>>>(p); break;
    }
    MC_LAUNCH_CHECK();
    return MC_OK;
  }
#define MC_DEC_CASE(A)                                              \
  case A:                                                           \
    note_launch();                                                  \
    if (sameb) k_decode_dense<A, true><<<grid, 256, 0, st>>>(p);    \
    else k_decode_dense<A, false><<<grid, 256, 0, st>>>(p);         \
    break;
  switch (s->algorithm) {
    MC_DEC_CASE(MC_IDENTITY)
    MC_DEC_CASE(MC_FP16)
    MC_DEC_CASE(MC_SIGNSGD)
    MC_DEC_CASE(MC_SIGNUM)
    MC_DEC_CASE(MC_EFSIGNSGD)
    MC_DEC_CASE(MC_ONEBIT)
    MC_DEC_CASE(MC_QSGD)
    MC_DEC_CASE(MC_TERNGRAD)
    MC_DEC_CASE(MC_INT8)
    default:
      set_error("decode_mean_dense: algorithm %d is not dense", s->algorithm);
      return MC_EINVAL;
  }
#undef MC_DEC_CASE
  MC_LAUNCH_CHECK();
  return MC_OK;
}

}  // namespace mc
