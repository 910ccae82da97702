// mc_sparse.cu — sparsifiers: topk / dgc_lite (radix select), threshold (stream
// compaction), randk (numpy Generator.choice restated on device), and the fused
// sparse decode + rank-ordered mean.
//
// Reference: _compress compressors.py:272-289, randk :278-285, EF :409-413, decode
// :439-448, aggregate :519-532.  Tie contract for top-k: among
// equal |x| at the k-th boundary the LOWEST indices are kept.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "mc_internal.cuh"

namespace mc {
namespace {

constexpr int TB = 256;         // threads per compaction block

// ------------------------------------------------------------------ workspace layout
// top-k radix select over the 31-bit magnitude key: 11 / 11 / 9 bits (a 12-bit first
// level measured no faster: the candidate list is not what bounds the later passes)
constexpr int H1B = 11, H2B = 11, H3B = 9;
constexpr int NB1 = 1 << H1B, NB2 = 1 << H2B, NB3 = 1 << H3B;
constexpr int S1 = 31 - H1B, S2 = S1 - H2B;
static_assert(S2 == H3B, "the three levels cover the 31-bit key");

struct SparseWS {
  uint32_t* keys;     // [n]  float bits of the corrected c32
  uint32_t* list;     // [n]  top-k: per-tile candidate segments (tile t's at its first element); randk scratch
  uint32_t* list2;    // [n]  top-k: the segments concatenated in order (the candidate list)
  uint32_t* segcnt;   // [ntiles + 1] top-k: candidates per pass-2 tile, then their exclusive prefix
  uint32_t* cmax;     // [ceil(n/128)] top-k: max |c32| key per 128-element chunk
  uint32_t* hist;     // [NB1 + NB2 + NB3] radix-select histograms (top-k)
  uint32_t* ctl;      // control words (see CTL_*)
  uint32_t* ticket;   // look-back ticket(s)
  uint64_t* status;   // look-back status [nblk]
  // randk
  uint32_t* draws;    // [k]   Floyd draws t_s
  uint32_t* htab;     // [2*H] hash (key, min step)
  uint32_t* bitmap;   // [ceil(n/32)]
  int64_t H;
  int64_t bytes;  // total workspace span (single source of truth for sparse_ws_bytes)
};
enum { CTL_B1 = 0, CTL_KREM1, CTL_B2, CTL_KREM2, CTL_T, CTL_NEED, CTL_M, CTL_GT, CTL_COUNT,
       CTL_DONE1, CTL_DONE2, CTL_DONE3, CTL_WORDS = 16 };

int64_t hash_size(int64_t k) {
  int64_t h = 1024;
  while (h < 4 * k) h <<= 1;
  return h;
}

SparseWS carve(uint8_t* w, int64_t n, int64_t k) {
  SparseWS s{};
  uint8_t* const w0 = w;
  const int64_t nblk = cdiv(n, 1024) + 1;  // finest look-back tiling in use (k_topk_final)
  s.keys = reinterpret_cast<uint32_t*>(w); w += a16(4 * n);
  s.list = reinterpret_cast<uint32_t*>(w); w += a16(4 * n);
  s.list2 = reinterpret_cast<uint32_t*>(w); w += a16(4 * n);
  s.segcnt = reinterpret_cast<uint32_t*>(w); w += a16(4 * (cdiv(n, 8192) + 1));
  s.cmax = reinterpret_cast<uint32_t*>(w); w += a16(4 * cdiv(n, 128));
  s.hist = reinterpret_cast<uint32_t*>(w); w += a16(4 * (NB1 + NB2 + NB3));
  s.ctl = reinterpret_cast<uint32_t*>(w); w += a16(4 * CTL_WORDS);
  s.ticket = reinterpret_cast<uint32_t*>(w); w += 16;
  s.status = reinterpret_cast<uint64_t*>(w); w += a16(8 * nblk);
  s.H = hash_size(k);
  s.draws = reinterpret_cast<uint32_t*>(w); w += a16(4 * k);
  s.htab = reinterpret_cast<uint32_t*>(w); w += a16(8 * s.H);
  s.bitmap = reinterpret_cast<uint32_t*>(w); w += a16(4 * cdiv(n, 32));
  s.bytes = (int64_t)(w - w0);
  return s;
}

// ------------------------------------------------------------------ block helpers
// Exclusive block scan of one uint64 per thread; returns exclusive prefix, *total = block sum.
__device__ __forceinline__ uint64_t block_exscan(uint64_t v, uint64_t* total) {
  __shared__ uint64_t s_w[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < nw ? s_w[lane] : 0, wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < nw) s_w[lane] = wi - w;
    if (lane == 31) s_w[31] = wi;  // nw <= 31 here (TB = 256)
  }
  __syncthreads();
  const uint64_t r = s_w[warp] + incl - v;
  *total = s_w[31];
  __syncthreads();
  return r;
}

__device__ __forceinline__ int64_t take_ticket(uint32_t* ticket) {
  __shared__ int64_t s_bid;
  if (threadIdx.x == 0) s_bid = atomicAdd(ticket, 1u);
  __syncthreads();
  return s_bid;
}

__device__ __forceinline__ uint64_t block_lookback(uint64_t* status, int64_t bid, uint64_t agg) {
  __shared__ uint64_t s_pre;
  if ((threadIdx.x >> 5) == 0) {
    const uint64_t pre = lookback_warp(status, bid, agg);
    if (threadIdx.x == 0) s_pre = pre;
  }
  __syncthreads();
  return s_pre;
}

// ------------------------------------------------------------------ top-k
// Radix select over the 31-bit magnitude key of c32 (|x| bits are monotone as u32):
//   pass1   EF prologue (r <- c in place), keys, 11-bit histogram; (fused N=1) out <- 0
//   select  bin B1 holding the k-th largest (one CTA)
//   pass2   ordered compaction (look-back) of every element with bin >= B1 into a list,
//           histogram of the next 11 bits of the bin-B1 candidates
//   select2 / hist3 / select3   resolve the exact threshold key T and the tie count
//   final   ordered filter of the list (key > T, or the first `need` ties = lowest
//           indices), EF fix-up r = c - c32 on the k survivors, (fused N=1) out[e] = c32
// Compaction kernels work on warp chunks of 1024 elements (lane holds 128 i + 4 lane + q,
// i < 8) so loads are coalesced 16-byte vectors; 8 warps = 8192 elements per tile.
constexpr int CW = 1024;
constexpr int CB = 8 * CW;

struct TP {
  Prologue pro;
  int64_t n, k;
  SparseWS w;
  uint32_t* err;
  uint32_t* idx_out;
  float* val_out;
  float* out;  // fused single-rank decode target (may alias g) or null
  int vec;
  int ksrc;  // where c32 lives after pass 1: KS_R (fp64 residual), KS_F (momentum or gradient), KS_KEYS
  const float* kf;
  uint8_t* payload;
  mc_payload_header hdr;
};
enum { KS_KEYS = 0, KS_R = 1, KS_F = 2 };

// float bits of element e's corrected c32 (pass 1 leaves it recoverable: the EF residual
// holds c, the momentum buffer / gradient holds w); keys are only materialised when the
// fused output would overwrite the gradient they come from
__device__ __forceinline__ uint32_t key_at(const TP& p, int64_t e) {
  if (p.ksrc == KS_R) return __float_as_uint(__double2float_rn(p.pro.r[e]));
  if (p.ksrc == KS_F) return __float_as_uint(p.kf[e]);
  return p.w.keys[e];
}

__device__ void select_bin(const uint32_t* hist, int nb, uint32_t k, uint32_t* out_bin, uint32_t* out_krem);

__global__ void __launch_bounds__(256) k_topk_pass1(TP p) {
  __shared__ uint32_t h[NB1];
  for (int i = threadIdx.x; i < NB1; i += blockDim.x) h[i] = 0;
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  bool bad = false;
  const int64_t groups = cdiv(p.n, 4);
  for (int64_t gi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < groups; gi += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e0 = 4 * gi;
    const bool full = p.vec && e0 + 3 < p.n;
    float x[4] = {0.0f, 0.0f, 0.0f, 0.0f}, mo[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    double rv[4] = {0.0, 0.0, 0.0, 0.0};
    if (full) {
      const float4 v = *reinterpret_cast<const float4*>(p.pro.g + e0);
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
      if (p.pro.m) {
        const float4 m = *reinterpret_cast<const float4*>(p.pro.m + e0);
        mo[0] = m.x; mo[1] = m.y; mo[2] = m.z; mo[3] = m.w;
      }
      if (p.pro.r) {
        const double2 a = *reinterpret_cast<const double2*>(p.pro.r + e0), b = *reinterpret_cast<const double2*>(p.pro.r + e0 + 2);
        rv[0] = a.x; rv[1] = a.y; rv[2] = b.x; rv[3] = b.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (e0 + q < p.n) {
          x[q] = p.pro.g[e0 + q];
          if (p.pro.m) mo[q] = p.pro.m[e0 + q];
          if (p.pro.r) rv[q] = p.pro.r[e0 + q];
        }
    }
    uint32_t key[4];
    double c[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool in = e0 + q < p.n;
      bad |= in && !isfinite(x[q]);
      float w = x[q];
      if (p.pro.m) {  // dgc accumulator b*m + x (two roundings, no FMA)  (compressors.py:405)
        w = p.pro.signum ? __fadd_rn(__fmul_rn(p.pro.beta, mo[q]), __fmul_rn(p.pro.omb, x[q]))
                         : __fadd_rn(__fmul_rn(p.pro.beta, mo[q]), x[q]);
        mo[q] = w;
      }
      c[q] = p.pro.r ? __dadd_rn((double)w, rv[q]) : (double)w;
      const float c32 = p.pro.r ? __double2float_rn(c[q]) : w;
      key[q] = __float_as_uint(c32);
      if (in) atomicAdd(&h[(key[q] & 0x7fffffffu) >> S1], 1u);
    }
    {  // the warp's 128 consecutive elements form one chunk: record their max magnitude key
      uint32_t km = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) km = max(km, (e0 + q < p.n) ? (key[q] & 0x7fffffffu) : 0u);
      km = __reduce_max_sync(__activemask(), km);
      if ((threadIdx.x & 31) == 0) p.w.cmax[e0 >> 7] = km;
    }
    if (full) {
      if (p.ksrc == KS_KEYS) *reinterpret_cast<uint4*>(p.w.keys + e0) = make_uint4(key[0], key[1], key[2], key[3]);
      if (p.pro.m) *reinterpret_cast<float4*>(p.pro.m + e0) = make_float4(mo[0], mo[1], mo[2], mo[3]);
      if (p.pro.r) {  // residual of unselected elements = c  (compressors.py:412)
        *reinterpret_cast<double2*>(p.pro.r + e0) = make_double2(c[0], c[1]);
        *reinterpret_cast<double2*>(p.pro.r + e0 + 2) = make_double2(c[2], c[3]);
      }
      if (p.out) *reinterpret_cast<float4*>(p.out + e0) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (e0 + q < p.n) {
          if (p.ksrc == KS_KEYS) p.w.keys[e0 + q] = key[q];
          if (p.pro.m) p.pro.m[e0 + q] = mo[q];
          if (p.pro.r) p.pro.r[e0 + q] = c[q];
          if (p.out) p.out[e0 + q] = 0.0f;
        }
    }
  }
  flag(p.err, bad, MC_ERR_NONFINITE);
  __syncthreads();
  for (int i = threadIdx.x; i < NB1; i += blockDim.x)
    if (h[i]) atomicAdd(&p.w.hist[i], h[i]);
  if (last_cta(&p.w.ctl[CTL_DONE1])) {  // select1: the bin holding the k-th largest
    __shared__ uint32_t s_b, s_r;
    select_bin(p.w.hist, NB1, (uint32_t)p.k, &s_b, &s_r);
    __syncthreads();
    if (threadIdx.x == 0) { p.w.ctl[CTL_B1] = s_b; p.w.ctl[CTL_KREM1] = s_r; }
  }
}

// find the bin holding the k-th largest: scans nb bins from the top (one CTA of 1024)
__device__ void select_bin(const uint32_t* hist, int nb, uint32_t k, uint32_t* out_bin, uint32_t* out_krem) {
  __shared__ uint32_t s_w[32];
  const int per = (nb + blockDim.x - 1) / blockDim.x;  // contiguous bins per thread, descending order
  const int t = threadIdx.x;
  uint32_t own = 0;
  for (int q = 0; q < per; ++q) {
    const int b = nb - t * per - 1 - q;
    if (b >= 0) own += hist[b];
  }
  const int lane = t & 31, warp = t >> 5;
  uint32_t incl = own;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_w[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = s_w[lane], wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(FULL, wi, o);
      if (lane >= o) wi += v;
    }
    s_w[lane] = wi - w;
  }
  __syncthreads();
  uint32_t run = s_w[warp] + incl - own;  // count in bins above my range
  for (int q = 0; q < per; ++q) {
    const int b = nb - t * per - 1 - q;
    if (b < 0) break;
    const uint32_t hb = hist[b];
    if (run < k && run + hb >= k) { *out_bin = (uint32_t)b; *out_krem = k - run; }
    run += hb;
  }
}


// Warp-chunk ordered compaction helper: given this lane's keep bits (bit 4 i + q for
// element 128 i + 4 lane + q of the warp chunk), returns this lane's base position for
// each i (within the warp chunk) and the warp total.
__device__ __forceinline__ uint32_t warp_chunk_offsets(uint32_t keep, uint32_t (&base)[8]) {
  const int lane = threadIdx.x & 31;
  uint32_t run = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t cnt = __popc((keep >> (4 * i)) & 0xfu);
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    base[i] = run + incl - cnt;
    run += __shfl_sync(FULL, incl, 31);
  }
  return run;
}

// CTA-level: exclusive prefix of the 8 warp totals + look-back over tiles.
__device__ __forceinline__ uint64_t cta_chunk_prefix(uint64_t warp_total, uint64_t* status, int64_t bid,
                                                     uint64_t& tile_total) {
  __shared__ uint64_t s_t[8];
  __shared__ uint64_t s_pre;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) s_t[warp] = warp_total;
  __syncthreads();
  uint64_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    before += (w < warp) ? s_t[w] : 0;
    tot += s_t[w];
  }
  if (warp == 0) {
    const uint64_t pre = lookback_warp(status, bid, tot);
    if (lane == 0) s_pre = pre;
  }
  __syncthreads();
  tile_total = tot;
  const uint64_t r = s_pre + before;
  __syncthreads();  // s_t / s_pre reused by the next tile
  return r;
}

// pass 2: one CTA per 8192-element tile compacts the tile's candidates (bin >= B1), in
// element order, into the tile's own segment of `list` (starting at the tile's first
// element, so it always fits) and records the count — no ordering between tiles (a
// look-back chain over 12K tiles costs more than the whole read).  Only 128-element chunks
// whose pass-1 maximum reaches bin B1 are read at all.
__global__ void __launch_bounds__(256) k_topk_pass2(TP p) {
  __shared__ uint32_t s_wt[8];
  const uint32_t B1 = p.w.ctl[CTL_B1], thr = B1 << S1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t bid = blockIdx.x;
  const int64_t nchunks = cdiv(p.n, 128);
  const int64_t c0 = bid * CB + (int64_t)warp * CW;
  const int64_t ch0 = c0 >> 7;  // this warp's 8 chunks
  const uint32_t cm = (lane < 8 && ch0 + lane < nchunks) ? p.w.cmax[ch0 + lane] : 0u;
  const uint32_t live = __ballot_sync(FULL, lane < 8 && ch0 + lane < nchunks && cm >= thr) & 0xffu;
  uint32_t kk[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t e0 = c0 + 128 * i + 4 * lane;
#pragma unroll
    for (int q = 0; q < 4; ++q) kk[i][q] = 0u;
    if (!((live >> i) & 1u)) continue;
    if (p.vec && e0 + 3 < p.n && p.ksrc != KS_KEYS) {
      if (p.ksrc == KS_R) {
        const double2 a = *reinterpret_cast<const double2*>(p.pro.r + e0), b = *reinterpret_cast<const double2*>(p.pro.r + e0 + 2);
        kk[i][0] = __float_as_uint(__double2float_rn(a.x)); kk[i][1] = __float_as_uint(__double2float_rn(a.y));
        kk[i][2] = __float_as_uint(__double2float_rn(b.x)); kk[i][3] = __float_as_uint(__double2float_rn(b.y));
      } else {
        const float4 v = *reinterpret_cast<const float4*>(p.kf + e0);
        kk[i][0] = __float_as_uint(v.x); kk[i][1] = __float_as_uint(v.y);
        kk[i][2] = __float_as_uint(v.z); kk[i][3] = __float_as_uint(v.w);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (e0 + q < p.n) kk[i][q] = key_at(p, e0 + q);
    }
  }
  uint32_t keep = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if (!((live >> i) & 1u)) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t key = kk[i][q] & 0x7fffffffu;
      const bool in = c0 + 128 * i + 4 * lane + q < p.n;
      keep |= (uint32_t)(in && key >= thr) << (4 * i + q);
      // the few keys inside bin B1 go straight to the L2 histogram (no per-tile smem copy)
      if (in && (key >> S1) == B1) atomicAdd(&p.w.hist[NB1 + ((key >> S2) & (NB2 - 1))], 1u);
    }
  }
  const uint32_t wtot = __reduce_add_sync(FULL, __popc(keep));
  if (lane == 0) s_wt[warp] = wtot;
  __syncthreads();
  uint32_t before = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    before += (w < warp) ? s_wt[w] : 0;
    tot += s_wt[w];
  }
  if (wtot) {
    uint32_t base[8];
    warp_chunk_offsets(keep, base);
    uint32_t* seg = p.w.list + bid * CB;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t pos = before + base[i];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (keep & (1u << (4 * i + q))) seg[pos++] = (uint32_t)(c0 + 128 * i + 4 * lane + q);
    }
  }
  if (threadIdx.x == 0) p.w.segcnt[bid] = tot;
}

// hist3: every CTA turns the pass-2 tile counts into their exclusive prefix in shared
// memory (one coalesced L2 read of ntiles words) and resolves select2 itself; then, grid-
// stride over list positions (a position's tile by binary search in smem, so one crowded
// tile does not serialise on one CTA), it concatenates the tile segments into list2 (the
// ordered candidate list) and histograms the low 9 key bits of the entries inside
// (B1, B2).  The last CTA resolves select3 (the exact threshold key T and the tie quota).
constexpr int64_t H3_MAX_TILES = 48 * 1024;  // 192 KB of prefix in smem: groups <= 402M elements
__global__ void __launch_bounds__(256) k_topk_hist3(TP p, int64_t ntiles) {
  extern __shared__ uint32_t pre[];  // [ntiles + 1]
  __shared__ uint32_t h3[NB3];
  __shared__ uint32_t s_b2, s_krem;
  for (int i = threadIdx.x; i < NB3; i += blockDim.x) h3[i] = 0;
  for (int64_t t = threadIdx.x; t < ntiles; t += blockDim.x) pre[t] = p.w.segcnt[t];
  select_bin(p.w.hist + NB1, NB2, p.w.ctl[CTL_KREM1], &s_b2, &s_krem);  // (ends in a barrier)
  __syncthreads();
  // exclusive scan in place: thread t owns a run of `per` consecutive tiles
  const int64_t per = cdiv(ntiles, 256);
  const int64_t t0 = threadIdx.x * per, t1 = imin(ntiles, t0 + per);
  uint64_t own = 0;
  for (int64_t t = t0; t < t1; ++t) own += pre[t];
  uint64_t total;
  uint64_t run = block_exscan(own, &total);  // (barriers: every thread has read its run)
  for (int64_t t = t0; t < t1; ++t) { const uint32_t c = pre[t]; pre[t] = (uint32_t)run; run += c; }
  if (threadIdx.x == 0) pre[ntiles] = (uint32_t)total;
  __syncthreads();
  const uint32_t M = (uint32_t)total;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.w.ctl[CTL_M] = M;  // list length
    p.w.ctl[CTL_B2] = s_b2;
    p.w.ctl[CTL_KREM2] = s_krem;
  }
  const uint32_t hi = (p.w.ctl[CTL_B1] << H2B) | s_b2;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < M; j += gridDim.x * blockDim.x) {
    int64_t lo = 0, up = ntiles;  // largest t with pre[t] <= j
    while (up - lo > 1) {
      const int64_t mid = (lo + up) >> 1;
      if (pre[mid] <= j) lo = mid; else up = mid;
    }
    const uint32_t e = p.w.list[lo * CB + (j - pre[lo])];
    p.w.list2[j] = e;
    const uint32_t key = key_at(p, e) & 0x7fffffffu;
    if ((key >> S2) == hi) atomicAdd(&h3[key & (NB3 - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB3; i += blockDim.x)
    if (h3[i]) atomicAdd(&p.w.hist[NB1 + NB2 + i], h3[i]);
  if (last_cta(&p.w.ctl[CTL_DONE3])) {
    __shared__ uint32_t s_b3, s_need;
    select_bin(p.w.hist + NB1 + NB2, NB3, p.w.ctl[CTL_KREM2], &s_b3, &s_need);
    __syncthreads();
    if (threadIdx.x == 0) {
      p.w.ctl[CTL_T] = (p.w.ctl[CTL_B1] << S1) | (p.w.ctl[CTL_B2] << S2) | s_b3;
      p.w.ctl[CTL_NEED] = s_need;
    }
  }
}

// final: persistent, ticketed tiles over the list; per element gt = key > T, tie = key == T.
// The packed (gt << 32 | tie) prefix gives slot = gt_before + min(tie_before, need).
// The list is short (k plus one histogram bin), so tiles are small (FI = 1: 1024 entries
// per CTA) to spread the random key reads over many SMs.
constexpr int FI = 1;
constexpr int CB_F = 8 * 128 * FI;

__global__ void __launch_bounds__(256) k_topk_final(TP p) {
  const uint32_t M = p.w.ctl[CTL_M], T = p.w.ctl[CTL_T], need = p.w.ctl[CTL_NEED];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  while (true) {
    const int64_t bid = take_ticket(p.w.ticket);
    if (bid * CB_F >= (int64_t)M) break;  // no later tile depends on an empty one
    const int64_t c0 = bid * CB_F + (int64_t)warp * 128 * FI;
    uint32_t gt = 0, tie = 0, ent[FI][4];
#pragma unroll
    for (int i = 0; i < FI; ++i)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t li = c0 + 128 * i + 4 * lane + q;
        ent[i][q] = 0;
        if (li < M) {
          const uint32_t e = p.w.list2[li];
          ent[i][q] = e;
          const uint32_t key = key_at(p, e) & 0x7fffffffu;
          gt |= (uint32_t)(key > T) << (4 * i + q);
          tie |= (uint32_t)(key == T) << (4 * i + q);
        }
      }
    // per-i warp scans of the packed counts (gt in the high half, ties in the low half)
    uint32_t base[FI];
    uint32_t run = 0;
#pragma unroll
    for (int i = 0; i < FI; ++i) {
      const uint32_t cnt = (__popc((gt >> (4 * i)) & 0xfu) << 16) | __popc((tie >> (4 * i)) & 0xfu);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
      }
      base[i] = run + incl - cnt;
      run += __shfl_sync(FULL, incl, 31);
    }
    const uint64_t wtot = ((uint64_t)(run >> 16) << 32) | (run & 0xffffu);
    uint64_t tile_total;
    const uint64_t pre = cta_chunk_prefix(wtot, p.w.status, bid, tile_total);
#pragma unroll
    for (int i = 0; i < FI; ++i) {
      uint64_t gt_b = (pre >> 32) + (base[i] >> 16), tie_b = (pre & 0xffffffffull) + (base[i] & 0xffffu);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t bit = 1u << (4 * i + q);
        const bool is_gt = gt & bit, is_tie = tie & bit;
        if (is_gt || (is_tie && tie_b < need)) {
          const uint64_t slot = gt_b + (tie_b < need ? tie_b : need);
          const uint32_t e = ent[i][q];
          const float c32 = __uint_as_float(key_at(p, e));
          p.idx_out[slot] = e;
          p.val_out[slot] = c32;
          if (p.pro.r) p.pro.r[e] = __dsub_rn(p.pro.r[e], (double)c32);  // r = c - decode  (:412)
          if (p.out) p.out[e] = __fadd_rn(0.0f, c32);                    // aggregate([payload])
        }
        gt_b += is_gt;
        tie_b += is_tie;
      }
    }
  }
}

// ------------------------------------------------------------------ threshold
struct ThP {
  Prologue pro;
  int64_t n;
  float tau;
  uint32_t* ticket;
  uint64_t* status;
  uint32_t* err;
  uint32_t* idx_out;
  float* val_out;
  float* out;  // fused single-rank decode (may alias g) or null
  int vec;
  int64_t ntiles;
  uint8_t* payload;
  mc_payload_header hdr;
};

// One pass: EF prologue, |c32| >= f32(tau) (compressors.py:288), EF residual, and the
// ordered compaction of (index, value) by warp chunks + decoupled look-back over tiles;
// (fused N=1) out = sel ? 0 + c32 : 0.
template <bool EF, bool MOM>
__global__ void __launch_bounds__(256) k_threshold(ThP p) {
  while (true) {
    const int64_t bid = take_ticket(p.ticket);
    if (bid >= p.ntiles) break;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t c0 = bid * CB + (int64_t)warp * CW;
    uint32_t keep = 0;
    float v[8][4];
    bool bad = false;
    // all loads of the chunk are issued before any store (the output may alias the input)
    double rv[EF ? 8 : 1][4];
    float mo[MOM ? 8 : 1][4];
  #pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t e0 = c0 + 128 * i + 4 * lane;
      if (p.vec && e0 + 3 < p.n) {
        const float4 g4 = *reinterpret_cast<const float4*>(p.pro.g + e0);
        v[i][0] = g4.x; v[i][1] = g4.y; v[i][2] = g4.z; v[i][3] = g4.w;
        if (MOM) {
          const float4 m4 = *reinterpret_cast<const float4*>(p.pro.m + e0);
          mo[MOM ? i : 0][0] = m4.x; mo[MOM ? i : 0][1] = m4.y; mo[MOM ? i : 0][2] = m4.z; mo[MOM ? i : 0][3] = m4.w;
        }
        if (EF) {
          const double2 a = *reinterpret_cast<const double2*>(p.pro.r + e0), b = *reinterpret_cast<const double2*>(p.pro.r + e0 + 2);
          rv[EF ? i : 0][0] = a.x; rv[EF ? i : 0][1] = a.y; rv[EF ? i : 0][2] = b.x; rv[EF ? i : 0][3] = b.y;
        }
      } else {
  #pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool in = e0 + q < p.n;
          v[i][q] = in ? p.pro.g[e0 + q] : 0.0f;
          if (MOM) mo[MOM ? i : 0][q] = in ? p.pro.m[e0 + q] : 0.0f;
          if (EF) rv[EF ? i : 0][q] = in ? p.pro.r[e0 + q] : 0.0;
        }
      }
    }
  #pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t e0 = c0 + 128 * i + 4 * lane;
      const bool full = p.vec && e0 + 3 < p.n;
      double rn[4];
      float o[4], mn[4];
  #pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool in = e0 + q < p.n;
        const float x = v[i][q];
        bad |= in && !isfinite(x);
        float w = x;
        if (MOM) {
          const float m0 = mo[MOM ? i : 0][q];
          w = p.pro.signum ? __fadd_rn(__fmul_rn(p.pro.beta, m0), __fmul_rn(p.pro.omb, x))
                           : __fadd_rn(__fmul_rn(p.pro.beta, m0), x);
          mn[q] = w;
        }
        const double c = EF ? __dadd_rn((double)w, rv[EF ? i : 0][q]) : (double)w;
        const float c32 = EF ? __double2float_rn(c) : w;
        const bool sel = in && fabsf(c32) >= p.tau;
        keep |= (uint32_t)sel << (4 * i + q);
        v[i][q] = c32;
        rn[q] = sel ? __dsub_rn(c, (double)c32) : c;  // r = c - decode (0 where dropped)
        o[q] = sel ? __fadd_rn(0.0f, c32) : 0.0f;
      }
      if (full) {
        if (MOM) *reinterpret_cast<float4*>(p.pro.m + e0) = make_float4(mn[0], mn[1], mn[2], mn[3]);
        if (EF) {
          *reinterpret_cast<double2*>(p.pro.r + e0) = make_double2(rn[0], rn[1]);
          *reinterpret_cast<double2*>(p.pro.r + e0 + 2) = make_double2(rn[2], rn[3]);
        }
        if (p.out) *reinterpret_cast<float4*>(p.out + e0) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
  #pragma unroll
        for (int q = 0; q < 4; ++q)
          if (e0 + q < p.n) {
            if (MOM) p.pro.m[e0 + q] = mn[q];
            if (EF) p.pro.r[e0 + q] = rn[q];
            if (p.out) p.out[e0 + q] = o[q];
          }
      }
    }
    flag(p.err, bad, MC_ERR_NONFINITE);
    uint32_t base[8];
    const uint32_t wtot = warp_chunk_offsets(keep, base);
    uint64_t tile_total;
    const uint64_t pos0 = cta_chunk_prefix(wtot, p.status, bid, tile_total);
  #pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t pos = (uint32_t)(pos0 + base[i]);
  #pragma unroll
      for (int q = 0; q < 4; ++q)
        if (keep & (1u << (4 * i + q))) {
          p.idx_out[pos] = (uint32_t)(c0 + 128 * i + 4 * lane + q);
          p.val_out[pos] = v[i][q];
          ++pos;
        }
    }
    if (bid == p.ntiles - 1 && threadIdx.x == 0) {
      mc_payload_header h = p.hdr;
      h.n_idx = h.n_val = (uint32_t)(pos0 + tile_total);
      *reinterpret_cast<mc_payload_header*>(p.payload) = h;
    }
  }
}

// ------------------------------------------------------------------ randk
// numpy Generator.choice(n, k, replace=False).  Draws: 32-bit words
// lo(W0), hi(W0), lo(W1), ... of Philox4x64 blocks; bounded(j) = Lemire with rejection.
struct RP {
  Prologue pro;
  int64_t n, k;
  uint64_t k0, k1;
  SparseWS w;
  uint32_t* err;
  uint32_t* idx_out;
  float* val_out;
  float scale;       // f32(n / k) when unbiased
  float* out;        // fused single-rank decode target (may alias g) or null
  int unbiased;
  int tail_shuffle;  // numpy's tail-shuffle branch (k > n//50 and n > 10000)
  uint8_t* payload;
  mc_payload_header hdr;
  const uint64_t* dkey;  // device-resident Philox key (graph capture) or null: (k0, k1)
  float band_sig;        // speculated entering offsets: expectation +- (band_sig sd + 16)
};
__device__ __forceinline__ Philox randk_philox(const RP& p) {
  return p.dkey ? Philox{p.dkey[0], p.dkey[1]} : Philox{p.k0, p.k1};
}

__device__ __forceinline__ uint32_t draw32(const Philox& ph, uint64_t pos) {
  uint64_t w[4];
  ph.block(pos >> 3, w);
  const unsigned q = (unsigned)(pos >> 1) & 3u;  // selects, not a dynamically indexed (local) array
  const uint64_t x = q == 0 ? w[0] : q == 1 ? w[1] : q == 2 ? w[2] : w[3];
  return (pos & 1) ? (uint32_t)(x >> 32) : (uint32_t)x;
}

__device__ __forceinline__ uint32_t hslot(uint32_t key, int64_t H) { return (key * 0x9E3779B1u) & (uint32_t)(H - 1); }

// Floyd's collision test needs, for every drawn value, the first step that drew it: every
// writer of a draw inserts (value -> min step) into the open-addressing table right away
// (order-independent: CAS on the key, atomicMin on the step)
__device__ __forceinline__ void rk_put(const RP& p, int64_t s, uint32_t v) {
  p.w.draws[s] = v;
  if (p.tail_shuffle) return;  // the tail shuffle keeps its own (position -> value) table
  uint32_t h = hslot(v, p.w.H);
  while (true) {
    const uint32_t prev = atomicCAS(&p.w.htab[2 * h], 0xffffffffu, v);
    if (prev == 0xffffffffu || prev == v) { atomicMin(&p.w.htab[2 * h + 1], (uint32_t)s); break; }
    h = (h + 1) & (uint32_t)(p.w.H - 1);
  }
}

// Lemire-32 rejection of numpy's bounded draw in [0, j] (random_bounded_uint64 ->
// buffered_bounded_lemire_uint32):  m = u32 * (j+1); reject iff lo32(m) < (2^32-(j+1)) % (j+1).
__device__ __forceinline__ bool lemire_reject(uint32_t w, uint64_t excl, uint32_t& val) {
  const uint64_t m = (uint64_t)w * excl;
  val = (uint32_t)(m >> 32);
  const uint32_t left = (uint32_t)m;
  if (left >= excl) return false;  // fast accept (the common case)
  return left < (uint32_t)((0x100000000ull - excl) % excl);  // excl may be 2^32 only via n = 2^32
}

__device__ __forceinline__ uint64_t step_range(const RP& p, int64_t s) {
  return p.tail_shuffle ? (uint64_t)(p.n - 1 - s) : (uint64_t)(p.n - p.k + s);
}

// One CTA walks the draw stream in windows of 1024 positions.  Step s consumes draws
// until Lemire accepts for range j_s, so position q serves step q - t(q) with t the
// rejections before q.  Per window every position evaluates 16 candidate offsets t0+d
// (warp ballots -> masks), each warp turns its masks into a transition table
// d_in -> d_out, one thread composes the 32 tables to get every warp's entering offset,
// and accepted positions emit draws[step].  A window is truncated at the first warp
// whose offset would leave the 16 candidates (more rejections than candidates).
constexpr int WD = 16;

// (1024 threads; every thread of the CTA calls it).  Walks positions [base0, pos_end) (pos_end a
// multiple of 32, or past the stream) from entering offset t00; returns the exit offset.
__device__ int64_t randk_walk_body(const RP& p, const uint32_t* words, int64_t nwords, int64_t base0, int64_t t00,
                                   int64_t pos_end) {
  __shared__ uint32_t smask[32][WD];
  __shared__ uint8_t sF[32][WD];
  __shared__ int s_enter[33];
  __shared__ int s_nw;
  __shared__ int64_t s_base, s_t0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Philox ph = randk_philox(p);
  if (tid == 0) { s_base = base0; s_t0 = t00; }
  __syncthreads();
  int64_t pf_pos = s_base + tid;  // prefetched word for the (likely) next window position
  uint32_t pf = pf_pos < nwords ? words[pf_pos] : draw32(ph, (uint64_t)pf_pos);
  while (true) {
    const int64_t base = s_base, t0 = s_t0;
    if (base - t0 >= p.k || base >= pos_end) break;  // every step has its draw / the range is walked
    const int64_t pos = base + tid;
    const uint32_t w32 = pos == pf_pos ? pf : (pos < nwords ? words[pos] : draw32(ph, (uint64_t)pos));
    pf_pos = pos + 1024;
    if (pf_pos < nwords) pf = words[pf_pos];
    else pf = draw32(ph, (uint64_t)pf_pos);
    // candidate d serves step s = pos - t0 - d with range excl_d = j_s + 1 = A + s (Floyd) or
    // A - s (tail shuffle).  Since lo32(w * excl_d) = lo32(w * excl_0) -+ d * w, the fast
    // accept test (left >= excl, i.e. no rejection possible) costs two integer ops per d;
    // the exact Lemire threshold is evaluated only for the rare candidates that fail it.
    const int64_t s0 = pos - t0;
    const uint32_t A = p.tail_shuffle ? (uint32_t)p.n : (uint32_t)(p.n - p.k + 1);
    const uint32_t ex0 = p.tail_shuffle ? A - (uint32_t)s0 : A + (uint32_t)s0;
    const uint32_t l0 = w32 * ex0;  // lo32 of the product
    const uint32_t dl = p.tail_shuffle ? w32 : (0u - w32);  // left_d = l0 + d * dl
    uint32_t hit = 0;  // bit d: candidate d may reject
#pragma unroll
    for (int d = 0; d < WD; ++d) {
      const uint32_t ex = p.tail_shuffle ? ex0 + d : ex0 - d;
      hit |= (uint32_t)((l0 + (uint32_t)d * dl) < ex) << d;
    }
    if (hit) {  // exact test for the candidates that can reject, with step validity
      uint32_t rejm = 0;
      for (uint32_t h = hit; h; h &= h - 1) {
        const int d = __ffs(h) - 1;
        const int64_t s = s0 - d;
        const uint32_t ex = p.tail_shuffle ? ex0 + d : ex0 - d;
        const uint32_t left = l0 + (uint32_t)d * dl;
        if (s >= 0 && s < p.k && left < (0u - ex) % ex) rejm |= 1u << d;  // (2^32 - ex) mod ex
      }
      hit = rejm;
    }
    // transpose: mask for candidate d = lanes whose bit d is set
#pragma unroll
    for (int d = 0; d < WD; ++d) {
      const unsigned mb = __ballot_sync(FULL, (hit >> d) & 1u);
      if (lane == 0) smask[warp][d] = mb;
    }
    __syncthreads();
    if (lane < WD) {  // transition table of this warp: entering offset d -> leaving offset
      int d = lane, from = 0;
      while (from < 32) {
        const uint32_t m = smask[warp][d] & (0xffffffffu << from);
        if (!m) break;
        from = __ffs(m);  // position after the rejection
        if (++d >= WD) { d = 255; break; }
      }
      sF[warp][lane] = (uint8_t)d;
    }
    __syncthreads();
    if (warp == 0) {
      // compose the 32 tables in warp order; identity tables (no rejection for any d, the
      // common case) leave the offset unchanged, so only the others are walked serially
      bool ident = true;
#pragma unroll
      for (int d = 0; d < WD; ++d) ident &= sF[lane][d] == d;
      unsigned todo = __ballot_sync(FULL, !ident);
      int d = 0, nw = 32, enter = 0;
      while (todo) {
        const int w = __ffs(todo) - 1;
        todo &= todo - 1;
        const int nd = sF[w][d];  // uniform smem read
        if (nd == 255) { nw = w; break; }
        d = nd;
        if (lane > w) enter = d;
      }
      s_enter[lane] = enter;  // entering offset of warp `lane` (valid for lane <= nw)
      if (lane == 0) {
        s_enter[32] = d;
        s_nw = (int)imin(nw, (pos_end - base) >> 5);  // stop at pos_end
      }
    }
    __syncthreads();
    const int nw = s_nw;
    if (nw == 0) {
      // > WD rejections inside one warp's 32 positions: walk them one by one (never seen in practice)
      if (tid == 0) {
        int64_t q = base, t = t0;
        for (int i = 0; i < 32 && q - t < p.k; ++i, ++q) {
          uint32_t v;
          const uint32_t w = q < nwords ? words[q] : draw32(ph, (uint64_t)q);
          if (lemire_reject(w, step_range(p, q - t) + 1, v)) ++t;
          else rk_put(p, q - t, v);
        }
        s_base = q;
        s_t0 = t;
      }
      __syncthreads();
      continue;
    }
    if (warp < nw) {
      // rejection positions of this warp along the true path, from its entering offset
      uint32_t R = 0;
      if (lane == 0) {
        int d = s_enter[warp], from = 0;
        while (from < 32) {
          const uint32_t m = smask[warp][d] & (0xffffffffu << from);
          if (!m) break;
          const int f = __ffs(m) - 1;
          R |= 1u << f;
          from = f + 1;
          ++d;
        }
      }
      R = __shfl_sync(FULL, R, 0);
      const int d = s_enter[warp] + __popc(R & ((1u << lane) - 1));
      const int64_t s = pos - t0 - d;
      if (!((R >> lane) & 1u) && s >= 0 && s < p.k) {
        uint32_t v;
        lemire_reject(w32, step_range(p, s) + 1, v);
        rk_put(p, s, v);
      }
    }
    __syncthreads();
    if (tid == 0) {
      s_base = base + 32 * nw;
      s_t0 = t0 + s_enter[nw];
    }
    __syncthreads();
  }
  const int64_t t_exit = s_t0;
  __syncthreads();  // before a next call's thread 0 rewrites s_base / s_t0
  return t_exit;
}

__global__ void __launch_bounds__(1024) k_randk_walk(RP p, const uint32_t* words, int64_t nwords) {
  randk_walk_body(p, words, nwords, 0, 0, INT64_MAX);
}

// ---- multi-SM draw walk ------------------------------------------------------------------
// The draw stream is cut into windows of WP = 1024 positions.  The offset t (rejections so
// far) at a window's start is unknown, but it is close to its expectation E_w (the sum of the
// per-draw rejection probabilities ((2^32 - excl) mod excl) / 2^32 before the window):
//   tables  one CTA per window evaluates the window for every entering offset t in
//           [L_w, L_w + dwin), centred on E_w, dwin = 2 (5 sd_w + 16) <= DW (rejection masks
//           for all offsets in smem, then one thread per candidate walks them) -> r_w(t);
//   link    groups of 16 windows compose their tables in parallel, the last CTA chains the
//           groups t_{g+1} = comp_g(t_g) and replays every window's exact entering offset;
//   emit    one CTA per window re-walks from its exact t_w and writes draws[step];
//   fallback if t_w ever leaves its window's range (a > 5 sd excursion, or a band capped at
//           DW), the link kernel's last CTA walks serially the windows outside their
//           ranges and resolves the others by their tables.
constexpr int WP = 1024;
// RX: most rejections one 1024-position window may hold (tables entries and the emit
// re-walk).  A draw for range excl is rejected with p < excl / 2^32, so a window averages
// up to 1024 n / 2^32 rejections (33 for a 138M-element group): RX = 32 / 64 / 96 by size
// DW (speculated entering offsets per window) is 512, or 1024 when the walk's drift is
// large: the offset's deviation from its expectation is a sum of Bernoulli rejections with
// sd ~ sqrt(k * (n - k/2) / 2^33) (149 for a 138M-element group at 1%), and a window range
// of +-DW/2 must cover it or the serial fallback takes over

struct WalkCtl {
  int64_t fail_base, fail_t0;  // fallback start (fail_base < 0: none)
  int64_t nwin_used;
};

__device__ __forceinline__ uint32_t excl_of(const RP& p, int64_t s) {
  return p.tail_shuffle ? (uint32_t)(p.n - s) : (uint32_t)(p.n - p.k + 1 + s);
}

// rejection test of position word w32 for step s (fast accept, then the exact threshold)
__device__ __forceinline__ bool rejects(const RP& p, uint32_t w32, int64_t s) {
  if (s < 0 || s >= p.k) return false;
  const uint32_t ex = excl_of(p, s);
  const uint32_t left = w32 * ex;
  return left < ex && left < (0u - ex) % ex;
}

// Mean and variance of the rejections before draw-stream position S (steps clamp(s, 0, k-1),
// as the windows count them): step s rejects with p = r / 2^32, r = 2^32 mod excl(s), and on a
// run of equal q = floor(2^32 / excl) the remainder falls by q per unit of excl, so the sums
// over a run are closed forms in (m, r_first, q) — a few runs cover the whole stream.
__device__ void randk_drift(const RP& p, int64_t S, double& mean, double& var) {
  const int64_t k = p.k, n = p.n, S1 = S < k ? S : k;
  mean = var = 0.0;
  if (S1 > 0) {
    // excl values of steps [0, S1): ascending n-k+1 .. (Floyd) or the top S1 values (tail shuffle)
    int64_t a = p.tail_shuffle ? n - S1 + 1 : n - k + 1;
    const int64_t b = p.tail_shuffle ? n : n - k + S1;
    const double T = 4294967296.0;
    while (a <= b) {
      const int64_t q = 0x100000000ll / a, e = imin(b, 0x100000000ll / q);
      const double m = (double)(e - a + 1), r0 = (double)(0x100000000ll - q * a), qd = (double)q;
      const double sj = m * (m - 1.0) / 2.0, sj2 = (m - 1.0) * m * (2.0 * m - 1.0) / 6.0;
      const double s1 = (m * r0 - qd * sj) / T;                                   // sum p
      const double s2 = (m * r0 * r0 - 2.0 * r0 * qd * sj + qd * qd * sj2) / (T * T);  // sum p^2
      mean += s1;
      var += s1 - s2;
      a = e + 1;
    }
  }
  if (S > k) {  // positions past the last step count it again
    const uint32_t ex = excl_of(p, k - 1);
    const double pl = (double)((0u - ex) % ex) * 0x1.0p-32;
    mean += (double)(S - k) * pl;
    var += (double)(S - k) * pl * (1.0 - pl);
  }
}

// Per-step scratch the later randk kernels need zeroed (bitmap, hash table, the emit's
// look-back ticket + status, the link kernel's CTA counter): cleared by the tables kernel's
// CTAs on their way, instead of three memset launches
struct RkInit {
  uint32_t* ts;  int64_t ts_words;  // ticket + status -> 0
  uint32_t* bm;  int64_t bm_words;  // bitmap -> 0
  uint32_t* ht;  int64_t ht_words;  // hash (key, step) -> 0xffffffff
  uint32_t* done;                   // k_randk_link's finished-CTA counter -> 0
};
__device__ __forceinline__ void fill_words(uint32_t* d, int64_t nw, uint32_t v, int64_t i0, int64_t stride) {
  // d is 16-byte aligned (carve); uint4 body, scalar tail
  const int64_t n4 = nw >> 2;
  for (int64_t i = i0; i < n4; i += stride) reinterpret_cast<uint4*>(d)[i] = make_uint4(v, v, v, v);
  for (int64_t i = 4 * n4 + i0; i < nw; i += stride) d[i] = v;
}

// 32 consecutive candidates' filter bits in three instructions each: left + (2^32 - exb)
// carries out exactly when left >= exb (no hit), and madc shifts that carry into the mask
// (m = 2 m + carry) — one integer-ALU op per candidate where compare + select + merge took
// three; the mask comes out MSB-first and inverted, hence the final brev / not.
// Returns bit j = (left_j < exb) for left_j = left + j dl; advances left by 32 dl.
__device__ __forceinline__ uint32_t filter32(uint32_t& left, uint32_t dl, uint32_t exb) {
  const uint32_t K = 0u - exb;
  uint32_t m = 0, t;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    asm("add.cc.u32 %0, %2, %3;\n\tmadc.lo.u32 %1, %1, 2, 0;" : "=r"(t), "+r"(m) : "r"(left), "r"(K));
    left += dl;
  }
  return ~__brev(m);
}

constexpr int HQ = 16;  // queued filter hits per thread (mean ~3.2 at 1% density)
// two 1024-thread CTAs per SM (<= 32 registers) when the smem allows it (DW = 512): the
// ~270-window grid of a 25M-element group is then one wave, not two
template <int DW, int RX>
__global__ void __launch_bounds__(1024, DW <= 512 ? 2 : 1) k_randk_tables(RP p, uint32_t* words, int64_t nwords, int64_t nwin, int64_t* Lw,
                               uint8_t* tables, RkInit ini) {
  extern __shared__ uint32_t masks[];  // [DW + RX][32], the hit queues [1024][HQ] u16, row summaries [DW + RX]
  uint16_t* hitq = reinterpret_cast<uint16_t*>(masks + (DW + RX) * 32);
  uint32_t* rownz = reinterpret_cast<uint32_t*>(hitq + 1024 * HQ);  // bit j: row c has a rejection in word j
  __shared__ int64_t s_L;
  __shared__ int s_dw;
  const int64_t w = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  __shared__ __align__(16) uint32_t s_w32[WP];
  const Philox ph = randk_philox(p);
  if (tid == 128) {
    // expected offset at the window start and its variance (closed form; they only centre and
    // size the speculated range — the chain checks it).  The range is +-(5 sd + 16), at most
    // DW: early windows, whose offset is still nearly deterministic, evaluate a few dozen
    // entering offsets instead of DW.  A > 5 sd excursion (p ~ 6e-7 per window) hands the rest
    // of the stream to the serial walker: slower, never wrong.  (Warp 4 computes this while
    // warps 0-3 generate the window's draw words.)
    double t, vv;
    randk_drift(p, w * WP, t, vv);
    const int half = (int)ceil((double)p.band_sig * sqrt(vv)) + 16;
    const int dw = (int)imin(DW, (int64_t)((2 * half + 31) / 32 * 32));
    const int64_t L = imax(0, (int64_t)floor(t) - dw / 2);
    s_L = L;
    s_dw = dw;
    Lw[w] = L;
  }
  if (tid < WP / 8) {  // the window's 1024 draw words: 128 Philox blocks, one per thread of warps 0-3
    uint64_t b[4];
    ph.block((uint64_t)(w * (WP / 8) + tid), b);
    const uint4 lo = make_uint4((uint32_t)b[0], (uint32_t)(b[0] >> 32), (uint32_t)b[1], (uint32_t)(b[1] >> 32));
    const uint4 hi = make_uint4((uint32_t)b[2], (uint32_t)(b[2] >> 32), (uint32_t)b[3], (uint32_t)(b[3] >> 32));
    reinterpret_cast<uint4*>(s_w32)[2 * tid] = lo;
    reinterpret_cast<uint4*>(s_w32)[2 * tid + 1] = hi;
    // kept for the emit's re-walk (nwords = every window position)
    reinterpret_cast<uint4*>(words + w * WP)[2 * tid] = lo;
    reinterpret_cast<uint4*>(words + w * WP)[2 * tid + 1] = hi;
  }
  {
    const int64_t gi = (int64_t)blockIdx.x * blockDim.x + tid, gs = (int64_t)gridDim.x * blockDim.x;
    fill_words(ini.ts, ini.ts_words, 0u, gi, gs);
    fill_words(ini.bm, ini.bm_words, 0u, gi, gs);
    fill_words(ini.ht, ini.ht_words, 0xffffffffu, gi, gs);
    if (gi == 0) *ini.done = 0u;
  }
  __syncthreads();
  const int64_t L = s_L;
  const int dwin = s_dw;
  const int64_t pos = w * WP + tid;
  const uint32_t w32 = s_w32[tid];
  for (int i = tid; i < (dwin + RX) * 32; i += blockDim.x) masks[i] = 0u;
  for (int i = tid; i < dwin + RX; i += blockDim.x) rownz[i] = 0u;
  __syncthreads();
  // candidate c serves step s = pos - L - c: lo32(w * excl) moves by -+w and excl by -+1 per
  // candidate, so the "may reject" filter (left < excl, p ~ excl / 2^32 < 1%) is two adds and a
  // compare; the few hits take the exact threshold test and set their bit in the shared
  // [candidate][warp] mask matrix
  const int64_t s0 = pos - L;
  const uint32_t ex0 = excl_of(p, s0);
  const int nc = dwin + RX;
  uint32_t left = w32 * ex0;
  const uint32_t dl = p.tail_shuffle ? w32 : (0u - w32);
  // the filter compares against the largest excl of the range (a superset of the exact
  // "left < excl_c"; the range moves excl by < 2^11 of ~2^25): branch-free, 32 candidates
  // per mask word, only the (rare) set bits are queued.  Hits are tested after the scan, all
  // lanes together: testing them inside the scan made every warp run the exact test (an
  // integer modulo) whenever any of its 32 lanes hit, not ~0.6% of the time
  const uint32_t exb = p.tail_shuffle ? ex0 + (uint32_t)nc : ex0;
  uint16_t* q = hitq + tid * HQ;
  int nh = 0;
  for (int c0 = 0; c0 < nc; c0 += 32) {
    uint32_t m = filter32(left, dl, exb);
    if (nc - c0 < 32) m &= (1u << (nc - c0)) - 1u;
    while (m) {
      const int c = c0 + __ffs(m) - 1;
      m &= m - 1;
      if (nh < HQ) q[nh++] = (uint16_t)c;
      else if (rejects(p, w32, s0 - c)) {  // (never in practice)
        atomicOr(&masks[c * 32 + warp], 1u << lane);
        atomicOr(&rownz[c], 1u << warp);
      }
    }
  }
  const int nmax = __reduce_max_sync(FULL, nh);
  for (int i = 0; i < nmax; ++i) {
    const int c = i < nh ? q[i] : 0;
    if (i < nh && rejects(p, w32, s0 - c)) {
      atomicOr(&masks[c * 32 + warp], 1u << lane);
      atomicOr(&rownz[c], 1u << warp);
    }
  }
  __syncthreads();
  if (tid < dwin) {  // walk entering with offset L + tid
    // the row summaries jump straight to the next mask word holding a rejection: a few shared
    // loads per rejection instead of a scan of all 32 words of every row on the path
    int d = tid, bit = 0;
    bool ok = true;
    while (bit < WP) {
      const int word = bit >> 5;
      uint32_t m = masks[d * 32 + word] & (0xffffffffu << (bit & 31));
      int wb = word;
      if (!m) {
        const uint32_t nz = word < 31 ? rownz[d] & (0xfffffffeu << word) : 0u;  // words after `word`
        if (!nz) break;  // no rejection left on row d: the walk stays on it to the window's end
        wb = __ffs(nz) - 1;
        m = masks[d * 32 + wb];
      }
      bit = wb * 32 + __ffs(m);  // position after the rejection
      if (++d >= dwin + RX || d - tid >= RX) { ok = false; break; }
    }
    tables[w * DW + tid] = ok ? (uint8_t)(d - tid) : (uint8_t)255;
  } else if (tid < DW) {
    tables[w * DW + tid] = (uint8_t)255;  // outside this window's range
  }
}

// chain, in two levels, one launch: windows are grouped by CG; CTA g composes its group's CG
// tables (staged in shared memory) into one table over the group's first window — thread e
// walks the group from entering offset L_g + e, recording every intermediate entering offset
// mid[w][e] (-1 once the walk left the range) and the exit comp[g][e].  The last CTA to
// finish (counter) runs the serial recurrence over groups on a shared-memory copy of comp
// (ngrp dependent shared loads), replays every window's exact entering offset in parallel
// (one mid lookup each -> tin[w]), and, if the chain ever left a window's speculated range,
// walks the rest of the stream itself (randk_walk_body: slower, never wrong).
constexpr int CG = 16;
constexpr int64_t RK_LINK_SMEM = 160 * 1024;  // largest staged comp copy (+ static smem <= 227 KB)
template <int DW>
__global__ void __launch_bounds__(1024) k_randk_link(RP p, const uint32_t* words, int64_t nwords, const int64_t* Lw,
                                                     const uint8_t* tables, int64_t nwin, int* comp, int* mid, int* tg,
                                                     int64_t* tin, WalkCtl* ctl, uint32_t* done, int stage_comp) {
  __shared__ __align__(16) uint8_t s_tab[CG * DW];
  __shared__ int s_L[CG];
  __shared__ bool s_last;
  extern __shared__ int s_dyn[];  // last CTA: group bases [ngrp], group entries [ngrp], comp as int16 relative
  const int tid = threadIdx.x;
  const int64_t ngrp = cdiv(nwin, CG);
  {
    const int64_t g = blockIdx.x, w0 = g * CG;
    const int nwg = (int)imin(CG, nwin - w0);
    const uint4* src4 = reinterpret_cast<const uint4*>(tables + w0 * DW);
    for (int i = tid; i < nwg * DW / 16; i += blockDim.x) reinterpret_cast<uint4*>(s_tab)[i] = src4[i];
    if (tid < nwg) s_L[tid] = (int)Lw[w0 + tid];
    __syncthreads();
    if (tid < DW) {
      int t = s_L[0] + tid;
      for (int w = 0; w < nwg; ++w) {
        mid[(w0 + w) * DW + tid] = t;
        if (t < 0) continue;
        const unsigned c = (unsigned)(t - s_L[w]);
        const int r = c < (unsigned)DW ? (int)s_tab[w * DW + c] : 255;
        t = (r == 255) ? -1 : t + r;  // -1: left the speculated range inside the group
      }
      comp[g * DW + tid] = t;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
  }
  // ---- the last CTA: every group's comp / mid is written
  __shared__ int s_ng, s_texit;
  __shared__ unsigned long long s_served, s_fail;
  __shared__ int64_t s_fb, s_ft0;
  int* s_Lg = s_dyn;
  int* s_tg = s_dyn + ngrp;
  int16_t* s_comp = reinterpret_cast<int16_t*>(s_dyn + 2 * ngrp);
  if (stage_comp) {
    for (int64_t g = tid; g < ngrp; g += blockDim.x) s_Lg[g] = (int)Lw[g * CG];
    __syncthreads();
    // four independent L2 loads in flight per thread
    for (int64_t i0 = tid; i0 < ngrp * DW; i0 += 4 * (int64_t)blockDim.x) {
      int c[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * (int64_t)blockDim.x;
        c[u] = i < ngrp * DW ? __ldcg(comp + i) : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + u * (int64_t)blockDim.x;
        if (i < ngrp * DW) s_comp[i] = (int16_t)(c[u] < 0 ? -1 : c[u] - s_Lg[i / DW]);  // < DW + CG RX: int16
      }
    }
    __syncthreads();
  }
  if (tid == 0) {  // serial over groups: ngrp dependent lookups
    int t = 0;
    int64_t g = 0;
    for (; g < ngrp; ++g) {
      if (stage_comp) s_tg[g] = t;
      else tg[g] = t;
      const int Lg = stage_comp ? s_Lg[g] : (int)Lw[g * CG];
      const unsigned c = (unsigned)(t - Lg);
      int nt = -1;
      if (c < (unsigned)DW) {
        if (stage_comp) {
          const int r = s_comp[g * DW + c];
          nt = r < 0 ? -1 : Lg + r;
        } else {
          nt = __ldcg(comp + g * DW + c);
        }
      }
      if (nt < 0) { ++g; break; }  // the failure lies inside this group: found below
      t = nt;
    }
    s_ng = (int)g;  // groups with a known entering offset
    s_texit = t;
    s_served = s_fail = (unsigned long long)nwin;
  }
  __syncthreads();
  // every window of those groups in parallel: its entering offset, the first window whose
  // steps are all served (nwin_used) and the first that leaves its range (serial hand-over)
  const int64_t nw = imin(nwin, (int64_t)s_ng * CG);
  for (int64_t w = tid; w < nw; w += blockDim.x) {
    const int64_t g = w / CG, w0 = g * CG;
    const int tgg = stage_comp ? s_tg[g] : tg[g];
    const unsigned e = (unsigned)(tgg - (stage_comp ? s_Lg[g] : (int)Lw[w0]));
    int t;
    if (e < (unsigned)DW) {
      t = __ldcg(mid + w * DW + e);
      if (t < 0) continue;  // past this group's failing window
    } else {
      if (w != w0) continue;  // the group is entered outside its range: fails at its first window
      t = tgg;
    }
    if (w * WP - (int64_t)t >= p.k) { atomicMin(&s_served, (unsigned long long)w); continue; }
    const unsigned c = (unsigned)(t - (int)Lw[w]);
    const int r = c < (unsigned)DW ? (int)tables[w * DW + c] : 255;
    if (r == 255) {  // at most one such window: the chain's first failure
      atomicMin(&s_fail, (unsigned long long)w);
      s_ft0 = t;
      continue;
    }
    tin[w] = t;
  }
  __syncthreads();
  if (tid == 0) {
    s_fb = -1;
    if (s_fail < s_served) {
      s_fb = (int64_t)s_fail * WP;
      ctl->nwin_used = (int64_t)s_fail;
    } else {
      ctl->nwin_used = (int64_t)s_served;
      if (s_served == (unsigned long long)nwin && nwin * WP - (int64_t)s_texit < p.k) {
        s_fb = nwin * WP;  // ran out of windows before every step was served
        s_ft0 = s_texit;
      }
    }
    ctl->fail_base = s_fb;
    ctl->fail_t0 = s_ft0;
  }
  __syncthreads();
  if (s_fb >= 0) {
    // the walk left a window's speculated range (a > 5 sd excursion, or a band capped at DW): walk
    // serially only the windows whose exact entering offset lies outside their band, and resolve
    // every other one by its table as soon as the walk is back inside (emit_draws then emits those;
    // the serially walked ones are marked tin = -1, their draws already written)
    __shared__ int64_t s_w, s_t;
    __shared__ int s_mode;
    if (tid == 0) { s_w = s_fb / WP; s_t = s_ft0; }
    __syncthreads();
    while (true) {
      if (tid == 0) {
        int64_t w = s_w, t = s_t;
        int mode = 0;  // 0: every step served; 1: walk window w serially; 2: walk past the last window
        while (true) {
          if (w * WP - t >= p.k) break;
          if (w >= nwin) { mode = 2; break; }
          const unsigned c = (unsigned)(t - (int)Lw[w]);
          const int r = c < (unsigned)DW ? (int)tables[w * DW + c] : 255;
          if (r == 255) { mode = 1; break; }
          tin[w] = t;
          t += r;
          ++w;
        }
        s_w = w;
        s_t = t;
        s_mode = mode;
      }
      __syncthreads();
      const int mode = s_mode;
      const int64_t w = s_w, t = s_t;
      __syncthreads();
      if (mode == 0) break;
      const int64_t tout = randk_walk_body(p, words, nwords, w * WP, t, mode == 1 ? (w + 1) * WP : INT64_MAX);
      if (tid == 0) {
        if (mode == 1) tin[w] = -1;
        s_w = w + 1;
        s_t = tout;
      }
      __syncthreads();
      if (mode == 2) break;
    }
    if (tid == 0) ctl->nwin_used = imin(s_w, nwin);
  }
}

template <int RX>
__global__ void __launch_bounds__(1024, 2) k_randk_emit_draws(RP p, const uint32_t* words, int64_t nwords,
                                                           const int64_t* tin, const WalkCtl* ctl) {
  __shared__ uint32_t smask[RX][32];
  __shared__ int s_enter[32];
  const int64_t w = blockIdx.x;
  if (w >= ctl->nwin_used) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t t0 = tin[w];
  if (t0 < 0) return;  // walked serially by the link kernel's fallback
  const int64_t pos = w * WP + tid;
  const uint32_t w32 = words[pos];  // written by the tables kernel for every window position
  for (int i = tid; i < RX * 32; i += blockDim.x) (&smask[0][0])[i] = 0u;
  __syncthreads();
  {  // rejection masks of offsets t0 + d: the tables kernel's two-op filter, exact test on hits
    const int64_t s0 = pos - t0;
    const uint32_t ex0 = excl_of(p, s0);
    const uint32_t dl = p.tail_shuffle ? w32 : (0u - w32);
    const uint32_t exb = p.tail_shuffle ? ex0 + (uint32_t)RX : ex0;
    uint32_t left = w32 * ex0;
    for (int c0 = 0; c0 < RX; c0 += 32) {
      uint32_t m = filter32(left, dl, exb);
      while (m) {
        const int d = c0 + __ffs(m) - 1;
        m &= m - 1;
        if (rejects(p, w32, s0 - d)) atomicOr(&smask[d][warp], 1u << lane);
      }
    }
  }
  __syncthreads();
  if (tid == 0) {  // entering offsets of the 32 warps along the true path (<= RX-1 rejections)
    int d = 0;
    for (int wi = 0; wi < 32; ++wi) {
      s_enter[wi] = d;
      int bit = 0;
      while (bit < 32) {
        const uint32_t m = smask[d][wi] & (0xffffffffu << bit);
        if (!m) break;
        bit = __ffs(m);
        ++d;
      }
    }
  }
  __syncthreads();
  uint32_t R = 0;  // rejection positions of this warp
  if (lane == 0) {
    int d = s_enter[warp], bit = 0;
    while (bit < 32) {
      const uint32_t m = smask[d][warp] & (0xffffffffu << bit);
      if (!m) break;
      const int f = __ffs(m) - 1;
      R |= 1u << f;
      bit = f + 1;
      ++d;
    }
  }
  R = __shfl_sync(FULL, R, 0);
  const int d = s_enter[warp] + __popc(R & ((1u << lane) - 1));
  const int64_t s = pos - t0 - d;
  if (!((R >> lane) & 1u) && s >= 0 && s < p.k) {
    uint32_t v;
    lemire_reject(w32, (uint64_t)excl_of(p, s), v);
    rk_put(p, s, v);
  }
}

__device__ __forceinline__ uint32_t first_step(const RP& p, uint32_t key) {
  uint32_t h = hslot(key, p.w.H);
  while (true) {
    const uint32_t k = p.w.htab[2 * h];
    if (k == key) return p.w.htab[2 * h + 1];
    h = (h + 1) & (uint32_t)(p.w.H - 1);
  }
}

// Floyd's final set: value(s) = collision(s) ? j_s : t_s with
// collision(s) = t_s drawn earlier  OR  (n-k <= t_s < j_s AND collision(t_s - (n-k))).
__global__ void k_randk_floyd_mark(RP p) {
  const uint32_t base = (uint32_t)(p.n - p.k);
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < p.k; s += (int64_t)gridDim.x * blockDim.x) {
    int64_t cur = s;
    bool coll = false;
    while (true) {
      const uint32_t t = p.w.draws[cur];
      if (first_step(p, t) != (uint32_t)cur) { coll = true; break; }
      if (t >= base && (int64_t)t < (int64_t)base + cur) { cur = t - base; continue; }
      break;
    }
    const uint32_t v = coll ? (uint32_t)(base + s) : p.w.draws[s];
    atomicOr(&p.w.bitmap[v >> 5], 1u << (v & 31));
  }
}

// numpy's tail shuffle (Fisher-Yates over positions n-1 .. first): single thread, the
// permuted positions tracked in the hash table (position -> value).  Rare path.
__global__ void k_randk_tail_shuffle(RP p) {
  const int64_t H = p.w.H;
  auto lookup = [&](uint32_t pos, bool create) -> uint32_t* {
    uint32_t h = hslot(pos, H);
    while (true) {
      const uint32_t k = p.w.htab[2 * h];
      if (k == pos) return &p.w.htab[2 * h + 1];
      if (k == 0xffffffffu) {
        if (!create) return nullptr;
        p.w.htab[2 * h] = pos;
        p.w.htab[2 * h + 1] = pos;
        return &p.w.htab[2 * h + 1];
      }
      h = (h + 1) & (uint32_t)(H - 1);
    }
  };
  for (int64_t s = 0; s < p.k; ++s) {
    const uint32_t i = (uint32_t)(p.n - 1 - s), j = p.w.draws[s];
    uint32_t* vi = lookup(i, true);
    uint32_t* vj = lookup(j, true);
    const uint32_t t = *vj;
    *vj = *vi;
    *vi = t;
    atomicOr(&p.w.bitmap[t >> 5], 1u << (t & 31));  // position i is final: data[i] = t
  }
}

// full selection (k == n): every index
__global__ void k_bitmap_all(RP p) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < cdiv(p.n, 32); w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rem = p.n - 32 * w;
    p.w.bitmap[w] = rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
  }
}

// Ordered compaction of the bitmap -> ascending indices and values, fused with one
// streaming pass over the CTA's 32768 elements that is also the encode prologue
// (compressors.py:381-413): non-finite check, momentum update, EF residual r = c - decode
// (c where not selected) and, for the fused single-rank sync, out = 0 + decode.  The draw
// walk never reads the gradient, so it is read once, here.  The CTA publishes its count for
// the look-back first, streams, stages its selected (offset, value) pairs in shared memory
// and resolves its output position only at the end — by then every predecessor has
// published, so nobody waits; the pairs then go out as coalesced rows.  A CTA selecting more
// than RK_STAGE elements (dense randk) resolves first and writes them from the bitmap before
// streaming (its values must be read before the pass overwrites the state).
constexpr int RKW = 2;  // bitmap words per emit thread: 16384-element tiles (finer tail balance)
constexpr int RK_STAGE = 2048;  // 1% randk stages ~330 per CTA; denser CTAs write from the bitmap
template <bool EF, bool MOM, bool VEC>
__device__ __forceinline__ void rk_stream(const RP& p, int64_t e_base, const uint32_t* s_words, const uint32_t* s_rank,
                                          uint16_t* s_off, float* s_val, bool stage, bool& bad) {
  const Prologue& pro = p.pro;
  if constexpr (!EF && !MOM && VEC) {
    // stateless codec on aligned buffers: U float4 groups of the gradient loaded before any is
    // processed (U loads in flight per thread: the pass is latency-bound at one; the output may
    // alias g, but every element is read before its own store and the groups are disjoint)
    constexpr int U = 4, NG = TB * RKW * 8;
    for (int i0 = threadIdx.x; i0 < NG; i0 += U * TB) {
      float4 gv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = e_base + 4 * (int64_t)(i0 + u * TB);
        gv[u] = (i0 + u * TB < NG && e + 3 < p.n) ? __ldcs(reinterpret_cast<const float4*>(pro.g + e))
                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u * TB;
        const int64_t e = e_base + 4 * (int64_t)i;
        if (i >= NG || e >= p.n) break;
        const uint32_t wd = s_words[i >> 3];
        const int sh = (i & 7) * 4;
        const uint32_t sel4 = (wd >> sh) & 0xfu;
        uint32_t rk = stage ? s_rank[i >> 3] + __popc(wd & ((1u << sh) - 1u)) : 0u;
        const bool full = e + 3 < p.n;
        float w[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
        if (!full)
          for (int q = 0; q < 4; ++q) w[q] = e + q < p.n ? pro.g[e + q] : 0.0f;
        float o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          bad |= !isfinite(w[q]);
          const bool sel = (sel4 >> q) & 1u;
          const float v = p.unbiased ? __fmul_rn(w[q], p.scale) : w[q];
          o[q] = sel ? __fadd_rn(0.0f, v) : 0.0f;
          if (stage && sel) {
            s_off[rk] = (uint16_t)(4 * i + q);
            s_val[rk] = v;
            ++rk;
          }
        }
        if (p.out) {
          if (full) *reinterpret_cast<float4*>(p.out + e) = make_float4(o[0], o[1], o[2], o[3]);
          else
            for (int q = 0; q < 4 && e + q < p.n; ++q) p.out[e + q] = o[q];
        }
      }
    }
    return;
  }
  for (int i = threadIdx.x; i < TB * RKW * 8; i += blockDim.x) {  // float4 groups, coalesced
    const int64_t e = e_base + 4 * (int64_t)i;
    if (e >= p.n) break;
    const uint32_t wd = s_words[i >> 3];
    const int sh = (i & 7) * 4;
    const uint32_t sel4 = (wd >> sh) & 0xfu;
    uint32_t rk = stage ? s_rank[i >> 3] + __popc(wd & ((1u << sh) - 1u)) : 0u;
    const bool full = VEC && e + 3 < p.n;
    float w[4];
    if (full) {
      const float4 gv = __ldcs(reinterpret_cast<const float4*>(pro.g + e));
      w[0] = gv.x; w[1] = gv.y; w[2] = gv.z; w[3] = gv.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = e + q < p.n ? pro.g[e + q] : 0.0f;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) bad |= !isfinite(w[q]);
    if (MOM) {
      float mo[4];
      if (full) {
        const float4 mv = *reinterpret_cast<const float4*>(pro.m + e);
        mo[0] = mv.x; mo[1] = mv.y; mo[2] = mv.z; mo[3] = mv.w;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) mo[q] = e + q < p.n ? pro.m[e + q] : 0.0f;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        w[q] = pro.signum ? __fadd_rn(__fmul_rn(pro.beta, mo[q]), __fmul_rn(pro.omb, w[q]))
                          : __fadd_rn(__fmul_rn(pro.beta, mo[q]), w[q]);
      if (full) *reinterpret_cast<float4*>(pro.m + e) = make_float4(w[0], w[1], w[2], w[3]);
      else
        for (int q = 0; q < 4 && e + q < p.n; ++q) pro.m[e + q] = w[q];
    }
    double rv[4] = {0.0, 0.0, 0.0, 0.0}, rn[4];
    if (EF) {
      if (full) {
        const double2 r0 = *reinterpret_cast<const double2*>(pro.r + e);
        const double2 r1 = *reinterpret_cast<const double2*>(pro.r + e + 2);
        rv[0] = r0.x; rv[1] = r0.y; rv[2] = r1.x; rv[3] = r1.y;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) rv[q] = e + q < p.n ? pro.r[e + q] : 0.0;
      }
    }
    float o[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double c = EF ? __dadd_rn((double)w[q], rv[q]) : (double)w[q];
      const float c32 = EF ? __double2float_rn(c) : w[q];
      const bool sel = (sel4 >> q) & 1u;
      const float v = p.unbiased ? __fmul_rn(c32, p.scale) : c32;
      if (EF) rn[q] = sel ? __dsub_rn(c, (double)v) : c;
      o[q] = sel ? __fadd_rn(0.0f, v) : 0.0f;
      if (stage && sel) {
        s_off[rk] = (uint16_t)(4 * i + q);
        s_val[rk] = v;
        ++rk;
      }
    }
    if (EF) {
      if (full) {
        *reinterpret_cast<double2*>(pro.r + e) = make_double2(rn[0], rn[1]);
        *reinterpret_cast<double2*>(pro.r + e + 2) = make_double2(rn[2], rn[3]);
      } else {
        for (int q = 0; q < 4 && e + q < p.n; ++q) pro.r[e + q] = rn[q];
      }
    }
    if (p.out) {
      if (full) *reinterpret_cast<float4*>(p.out + e) = make_float4(o[0], o[1], o[2], o[3]);
      else
        for (int q = 0; q < 4 && e + q < p.n; ++q) p.out[e + q] = o[q];
    }
  }
}

template <bool EF, bool MOM, bool VEC>
// Persistent: a grid of (SMs x resident CTAs) takes tiles in ticket order until all are done
// (a tile waits in its look-back only on tiles whose tickets were taken earlier, by resident
// CTAs), so the last partial wave of a 782-tile ResNet-50 grid does not idle most SMs.
__global__ void __launch_bounds__(TB) k_randk_emit(RP p, int64_t ntiles) {
  __shared__ uint32_t s_words[TB * RKW], s_rank[TB * RKW];
  __shared__ uint16_t s_off[RK_STAGE];
  __shared__ float s_val[RK_STAGE];
  __shared__ uint64_t s_pre;
  bool bad = false;
  for (;;) {
  const int64_t bid = take_ticket(p.w.ticket);
  if (bid >= ntiles) break;
  if (bid == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  const int64_t nw = cdiv(p.n, 32);
  const int64_t w0 = bid * TB * RKW + (int64_t)threadIdx.x * RKW;  // RKW words (32 RKW elements) per thread
  uint32_t words[RKW];
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < RKW; ++q) {
    words[q] = (w0 + q < nw) ? p.w.bitmap[w0 + q] : 0u;
    cnt += __popc(words[q]);
  }
  uint64_t total;
  const uint64_t ex = block_exscan(cnt, &total);
  {
    uint32_t rk = (uint32_t)ex;
#pragma unroll
    for (int q = 0; q < RKW; ++q) {
      s_words[threadIdx.x * RKW + q] = words[q];
      s_rank[threadIdx.x * RKW + q] = rk;
      rk += __popc(words[q]);
    }
  }
  const int64_t e_base = bid * TB * RKW * 32;
  const bool stage = total <= RK_STAGE;
  if (stage) {
    if (threadIdx.x == 0) st_volatile(&p.w.status[bid], (bid == 0 ? LB_PRE : LB_AGG) | total);  // early
    __syncthreads();
    rk_stream<EF, MOM, VEC>(p, e_base, s_words, s_rank, s_off, s_val, true, bad);
    if ((threadIdx.x >> 5) == 0) {
      const uint64_t pre = lookback_warp(p.w.status, bid, total);
      if (threadIdx.x == 0) s_pre = pre;
    }
    __syncthreads();
    const uint64_t pre = s_pre;
    for (int j = threadIdx.x; j < (int)total; j += blockDim.x) {
      p.idx_out[pre + j] = (uint32_t)(e_base + s_off[j]);
      p.val_out[pre + j] = s_val[j];
    }
  } else {
    const uint64_t pre = block_lookback(p.w.status, bid, total);
    uint64_t pos = pre + ex;
#pragma unroll
    for (int q = 0; q < RKW; ++q) {
      uint32_t m = words[q];
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const int64_t e = (w0 + q) * 32 + b;
        float c32;
        p.pro.load(e, c32, bad, false);  // the state is written by the streaming pass below
        p.idx_out[pos] = (uint32_t)e;
        p.val_out[pos] = p.unbiased ? __fmul_rn(c32, p.scale) : c32;
        ++pos;
      }
    }
    __syncthreads();  // every selected value was read before the pass overwrites the state
    rk_stream<EF, MOM, VEC>(p, e_base, s_words, s_rank, s_off, s_val, false, bad);
  }
  __syncthreads();  // the tile's shared state (ticket, words, staging) is reused by the next one
  }
  flag(p.err, bad, MC_ERR_NONFINITE);
}

// ------------------------------------------------------------------ sparse decode-mean
struct SD {
  const uint8_t* base;
  int64_t stride;
  int nranks;
  int64_t n, ntiles;
  uint32_t* starts;  // [nranks][ntiles+1]
  float* out;
  uint32_t* err;
  uint32_t algo;
};
constexpr int DT = 8192;  // output tile (elements, 32 KB of smem)

__device__ __forceinline__ void sparse_sections(const uint8_t* pl, const uint32_t*& idx, const float*& val, uint32_t& cnt) {
  const mc_payload_header* h = reinterpret_cast<const mc_payload_header*>(pl);
  cnt = h->n_idx;
  idx = reinterpret_cast<const uint32_t*>(pl + HDR);
  val = reinterpret_cast<const float*>(pl + HDR + a16(4 * (int64_t)h->cap));
}

// per (rank, entry): tile start table + validation (range / strictly increasing)
__global__ void k_sparse_starts(SD p) {
  const int r = blockIdx.y;
  const uint8_t* pl = p.base + p.stride * r;
  const mc_payload_header* h = reinterpret_cast<const mc_payload_header*>(pl);
  const uint32_t* idx;
  const float* val;
  uint32_t cnt;
  sparse_sections(pl, idx, val, cnt);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (h->algorithm != p.algo || h->original_len != (uint64_t)p.n || cnt > h->cap || h->n_val != cnt)
      atomicOr(p.err, MC_ERR_HEADER);
  }
  uint32_t* st = p.starts + (int64_t)r * (p.ntiles + 1);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= cnt; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo, hi;
    if (e < cnt) {
      const uint32_t v = idx[e];
      if ((int64_t)v >= p.n) atomicOr(p.err, MC_ERR_INDEX_RANGE);
      if (e > 0 && idx[e - 1] >= v) atomicOr(p.err, MC_ERR_INDEX_ORDER);
      hi = imin(v / DT, p.ntiles);
      lo = e == 0 ? 0 : imin(idx[e - 1] / DT, p.ntiles) + 1;
    } else {
      hi = p.ntiles;
      lo = cnt == 0 ? 0 : imin(idx[cnt - 1] / DT, p.ntiles) + 1;
    }
    for (int64_t t = lo; t <= hi; ++t) st[t] = (uint32_t)e;
  }
}

__global__ void __launch_bounds__(256) k_sparse_tiles(SD p) {
  __shared__ __align__(16) float acc[DT];
  const int64_t t = blockIdx.x;
  const int64_t t0 = t * DT;
  for (int i = threadIdx.x; i < DT / 4; i += blockDim.x)
    reinterpret_cast<float4*>(acc)[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  __syncthreads();
  for (int r = 0; r < p.nranks; ++r) {
    const uint8_t* pl = p.base + p.stride * r;
    const uint32_t* idx;
    const float* val;
    uint32_t cnt;
    sparse_sections(pl, idx, val, cnt);
    const uint32_t* st = p.starts + (int64_t)r * (p.ntiles + 1);
    const uint32_t a = st[t], b = st[t + 1];
    for (uint32_t e = a + threadIdx.x; e < b; e += blockDim.x) {
      const int64_t off = (int64_t)idx[e] - t0;
      if (off >= 0 && off < DT) acc[off] = __fadd_rn(acc[off], val[e]);  // rank-ordered fp32 sum
    }
    __syncthreads();
  }
  const float fn = (float)p.nranks;
  // power-of-two rank counts: the exact reciprocal product equals the IEEE quotient
  const bool pow2 = (p.nranks & (p.nranks - 1)) == 0;
  const float inv = __fdiv_rn(1.0f, fn);
  auto mean = [&](float v) { return pow2 ? __fmul_rn(v, inv) : __fdiv_rn(v, fn); };
  const int64_t lim = imin(DT, p.n - t0);
  if (lim == DT && ((uintptr_t)(p.out + t0) % 16) == 0) {
    for (int i = threadIdx.x; i < DT / 4; i += blockDim.x) {
      const float4 v = reinterpret_cast<const float4*>(acc)[i];
      reinterpret_cast<float4*>(p.out + t0)[i] = make_float4(mean(v.x), mean(v.y), mean(v.z), mean(v.w));
    }
  } else {
    for (int i = threadIdx.x; i < lim; i += blockDim.x) p.out[t0 + i] = mean(acc[i]);
  }
}

}  // namespace

int64_t sparse_ws_bytes(const mc_spec* s, int64_t n) {
  const int64_t k = s->algorithm == MC_THRESHOLD ? 1 : top_k_count(s->sparsity, n);
  return carve(nullptr, n, k).bytes + 64;
}

static Prologue make_prologue(const EncodeArgs& a) {
  Prologue pro{};
  pro.g = a.g;
  pro.r = a.spec->error_feedback ? a.r : nullptr;
  pro.m = a.spec->has_momentum ? a.m : nullptr;
  pro.beta = a.spec->momentum;
  const float beta = a.spec->momentum;
  pro.omb = 1.0f - beta;  // np.float32(1.0) - coef: one f32 rounding (SSE, no excess precision)
  pro.signum = a.spec->algorithm == MC_SIGNUM;
  return pro;
}

int encode_topk(const EncodeArgs& a, float* out) {
  const int64_t n = a.n, k = top_k_count(a.spec->sparsity, n);
  TP p{};
  p.pro = make_prologue(a);
  p.n = n;
  p.k = k;
  p.w = carve(a.ws, n, k);
  p.err = a.ctx.err;
  p.idx_out = reinterpret_cast<uint32_t*>(a.payload + a.L.off_idx);
  p.val_out = reinterpret_cast<float*>(a.payload + a.L.off_val);
  p.out = out;
  p.vec = ((uintptr_t)p.pro.g % 16 == 0) && (!p.pro.r || (uintptr_t)p.pro.r % 16 == 0) &&
          (!p.pro.m || (uintptr_t)p.pro.m % 16 == 0) && ((uintptr_t)out % 16 == 0);
  p.payload = a.payload;
  // c32 after pass 1: f32(r) under EF, else the updated momentum, else the gradient — unless
  // the fused output (zeroed by pass 1) aliases that gradient: then keys are materialised
  if (p.pro.r) p.ksrc = KS_R;
  else if (p.pro.m) { p.ksrc = KS_F; p.kf = p.pro.m; }
  else if (out != p.pro.g) { p.ksrc = KS_F; p.kf = p.pro.g; }
  else p.ksrc = KS_KEYS;
  p.hdr.algorithm = (uint32_t)a.spec->algorithm;
  p.hdr.original_len = (uint64_t)n;
  p.hdr.n_idx = p.hdr.n_val = p.hdr.cap = (uint32_t)k;
  cudaStream_t st = a.ctx.stream;
  const int64_t ntiles = cdiv(n, CB);
  if (ntiles > H3_MAX_TILES) {
    set_error("top-k group of %lld elements exceeds the supported %lld", (long long)n, (long long)(H3_MAX_TILES * CB));
    return MC_EINVAL;
  }
  // one memset for the histograms, control words, and the final pass's ticket + look-back
  // status (passes 1-3 use neither ticket nor status)
  const int64_t ftiles = cdiv(n, CB_F);
  const size_t zbytes = (size_t)((uint8_t*)p.w.status - (uint8_t*)p.w.hist) + 8 * (imax(ntiles, ftiles) + 1);
  MC_API_CHECK(cudaMemsetAsync(p.w.hist, 0, zbytes, st));
  const unsigned g1 = (unsigned)imax(1, imin(cdiv(n, 1024), (int64_t)sm_count() * 8));
  note_launch(); k_topk_pass1<<<g1, 256, 0, st>>>(p);
  note_launch(); k_topk_pass2<<<(unsigned)ntiles, 256, 0, st>>>(p);
  const int h3smem = (int)(4 * (ntiles + 1));
  static std::atomic<uint64_t> h3_cfg{0};  // per device: the opt-in (to the largest table) is set
  if (h3smem > 48 * 1024) MC_API_CHECK(smem_optin(h3_cfg, k_topk_hist3, 4 * (int)(H3_MAX_TILES + 1)));
  note_launch(); k_topk_hist3<<<(unsigned)sm_count() * 2, 256, h3smem, st>>>(p, ntiles);
  note_launch(); k_topk_final<<<(unsigned)imax(1, imin(ftiles, (int64_t)sm_count() * 4)), 256, 0, st>>>(p);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int encode_threshold(const EncodeArgs& a, float* out) {
  const int64_t n = a.n;
  ThP p{};
  p.pro = make_prologue(a);
  p.n = n;
  p.tau = (float)a.spec->threshold;  // numpy 2 demotes the python float to f32 (NEP 50)
  SparseWS w = carve(a.ws, n, 1);
  p.ticket = w.ticket;
  p.status = w.status;
  p.err = a.ctx.err;
  p.idx_out = reinterpret_cast<uint32_t*>(a.payload + a.L.off_idx);
  p.val_out = reinterpret_cast<float*>(a.payload + a.L.off_val);
  p.payload = a.payload;
  p.hdr.algorithm = MC_THRESHOLD;
  p.hdr.original_len = (uint64_t)n;
  p.hdr.cap = (uint32_t)a.L.cap;
  p.out = out;
  p.vec = ((uintptr_t)p.pro.g % 16 == 0) && (!p.pro.r || (uintptr_t)p.pro.r % 16 == 0) &&
          (!p.pro.m || (uintptr_t)p.pro.m % 16 == 0) && ((uintptr_t)out % 16 == 0);
  const int64_t nblk = cdiv(n, CB);
  p.ntiles = nblk;
  cudaStream_t st = a.ctx.stream;
  MC_API_CHECK(cudaMemsetAsync(w.ticket, 0, 16 + 8 * (nblk + 1), st));
  const unsigned pgrid = (unsigned)imax(1, imin(nblk, (int64_t)sm_count() * 2));
  note_launch();
  if (p.pro.r) {
    if (p.pro.m) k_threshold<true, true><<<pgrid, 256, 0, st>>>(p);
    else k_threshold<true, false><<<pgrid, 256, 0, st>>>(p);
  } else {
    if (p.pro.m) k_threshold<false, true><<<pgrid, 256, 0, st>>>(p);
    else k_threshold<false, false><<<pgrid, 256, 0, st>>>(p);
  }
  MC_LAUNCH_CHECK();
  return MC_OK;
}

struct RandkStats {
  double sd, window_mean_max;
};
// Lemire rejection probability of step s is ((2^32 - excl) mod excl) / 2^32 = 1 - q excl / 2^32
// with q = floor(2^32 / excl): linear in excl on every run of equal q (a sawtooth).  The k
// steps cover excl in [lo, lo + k), so the sums over each run are closed forms — the variance
// of the walk's drift and the largest mean rejection count of a 1024-step window (piecewise
// linear in the window start: maximal where a window starts or ends at a run boundary) in
// O(number of runs), no per-step loop and no cache.
RandkStats randk_stats(int64_t n, int64_t k, bool tail_shuffle) {
  const long double T = 4294967296.0L;
  (void)tail_shuffle;  // Floyd walks excl = n-k+1 .. n upwards, the tail shuffle n .. n-k+1 down:
  const int64_t lo = n - k + 1, hi = n;  // the same values, and the same set of 1024-step windows
  auto q_of = [](int64_t e) { return (int64_t)(0x100000000ll / e); };
  // sum of p over excl in [a, b] (one run of constant q), and of p^2
  auto run_sums = [&](int64_t a, int64_t b, int64_t q, long double& s1, long double& s2) {
    const long double m = (long double)(b - a + 1), se = ((long double)a + b) * m / 2.0L;
    auto sq = [](long double x) { return x * (x + 1) * (2 * x + 1) / 6.0L; };
    const long double se2 = sq((long double)b) - sq((long double)a - 1);
    s1 = (m * T - q * se) / T;
    s2 = (m * T * T - 2.0L * T * q * se + (long double)q * q * se2) / (T * T);
  };
  std::vector<int64_t> bnd;  // run starts in [lo, hi]
  long double var = 0.0L;
  for (int64_t a = lo; a <= hi;) {
    const int64_t q = q_of(a), b = imin(hi, 0x100000000ll / q);  // last excl with the same q
    long double s1, s2;
    run_sums(a, b, q, s1, s2);
    var += s1 - s2;
    bnd.push_back(a);
    a = b + 1;
  }
  // window sum over excl [x, x + W) via runs
  auto wsum = [&](int64_t x) {
    const int64_t y = imin(hi, x + WP - 1);
    long double t = 0.0L;
    for (int64_t a = x; a <= y;) {
      const int64_t q = q_of(a), b = imin(y, 0x100000000ll / q);
      long double s1, s2;
      run_sums(a, b, q, s1, s2);
      t += s1;
      a = b + 1;
    }
    return (double)t;
  };
  // breakpoints of the window start x: x or x + WP - 1 on a run boundary
  double best = std::max(wsum(lo), wsum(imax(lo, hi - WP + 1)));
  for (int64_t r : bnd)
    for (int64_t x : {r, r - WP, r - WP + 1})
      if (x >= lo && x <= hi) best = std::max(best, wsum(x));
  return RandkStats{sqrt((double)var), best};
}

// persistent grid of the emit: every resident CTA slot (occupancy queried once per kernel)
template <typename K>
unsigned rk_grid(K* kernel, int64_t ntiles) {
  static std::atomic<int> occ{0};
  int o = occ.load(std::memory_order_relaxed);
  if (o == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kernel, TB, 0) != cudaSuccess || o < 1) o = 1;
    occ.store(o, std::memory_order_relaxed);
  }
  return (unsigned)imax(1, imin(ntiles, (int64_t)sm_count() * o));
}

int encode_randk(const EncodeArgs& a, float* out) {
  const int64_t n = a.n, k = top_k_count(a.spec->sparsity, n);
  RP p{};
  p.pro = make_prologue(a);
  p.n = n;
  p.k = k;
  p.k0 = a.k0;
  p.k1 = a.k1;
  p.dkey = a.dkey;
  p.w = carve(a.ws, n, k);
  p.err = a.ctx.err;
  p.idx_out = reinterpret_cast<uint32_t*>(a.payload + a.L.off_idx);
  p.val_out = reinterpret_cast<float*>(a.payload + a.L.off_val);
  p.unbiased = a.spec->unbiased_scaling;
  p.scale = (float)((double)n / (double)k);  // np.float32(n / k)  (compressors.py:284)
  p.tail_shuffle = (n > 10000 && k > n / 50) ? 1 : 0;
  {  // MC_RANDK_BAND_SIGMA: test knob (a narrow band forces the serial fallback; results never change)
    const char* e = getenv("MC_RANDK_BAND_SIGMA");
    p.band_sig = e ? (float)atof(e) : 5.0f;  // +-5 sd: an excursion past it (p ~ 6e-7 per window) only costs time
  }
  p.out = out;
  p.payload = a.payload;
  p.hdr.algorithm = MC_RANDK;
  p.hdr.flags = p.unbiased ? 1u : 0u;
  p.hdr.original_len = (uint64_t)n;
  p.hdr.n_idx = p.hdr.n_val = p.hdr.cap = (uint32_t)k;
  cudaStream_t st = a.ctx.stream;
  const int64_t nwords = cdiv(n, 32);
  const int64_t nblk = cdiv(nwords, TB * RKW) + 1;
  const bool vec = (uintptr_t)p.pro.g % 16 == 0 && (!out || (uintptr_t)out % 16 == 0) &&
                   (!p.pro.r || (uintptr_t)p.pro.r % 16 == 0) && (!p.pro.m || (uintptr_t)p.pro.m % 16 == 0);
  auto memsets = [&]() -> int {
    MC_API_CHECK(cudaMemsetAsync(p.w.ticket, 0, 16 + 8 * (nblk + 1), st));
    MC_API_CHECK(cudaMemsetAsync(p.w.bitmap, 0, 4 * nwords, st));
    MC_API_CHECK(cudaMemsetAsync(p.w.htab, 0xff, 8 * p.w.H, st));
    return MC_OK;
  };
  if (k == n) {
    if (int rc = memsets()) return rc;
    note_launch(); k_bitmap_all<<<(unsigned)imax(1, imin(cdiv(nwords, 256), 1024)), 256, 0, st>>>(p);
  } else {
    // the 32-bit draw stream (k + margin for rejections) in the unused candidate-list area;
    // walk scratch after it: L_w, entering offsets, control, tables, composed tables
    const int64_t ndraw = imin(n, k + k / 16 + 4096);
    const int64_t nwin = cdiv(ndraw, WP);
    const int64_t nwpos = nwin * WP;  // draw words kept for every window position
    uint8_t* wsb = reinterpret_cast<uint8_t*>(p.w.list) + a16(4 * nwpos);
    int64_t* Lw = reinterpret_cast<int64_t*>(wsb + a16(16 * nwin));
    int64_t* tin = reinterpret_cast<int64_t*>(wsb + a16(16 * nwin) + a16(8 * nwin));
    WalkCtl* ctl = reinterpret_cast<WalkCtl*>(wsb + a16(16 * nwin) + 2 * a16(8 * nwin));
    uint8_t* tables = wsb + a16(16 * nwin) + 2 * a16(8 * nwin) + 64;
    // exact drift statistics of this (n, k) stream: sd of the total rejections and the largest
    // mean rejection count of a 1024-draw window
    const RandkStats rs = randk_stats(n, k, p.tail_shuffle != 0);
    const int DWr = rs.sd > 100.0 ? 1024 : 512;  // +-256 covers >= 2.56 sd; the rest falls back
    const double mu = rs.window_mean_max;
    auto tail = [&](int r) {  // P(Poisson(mu) >= r) over all windows
      double term = exp(-mu), sum = 0.0;
      for (int j = 1; j <= r; ++j) term *= mu / j;
      for (int j = r; j < r + 400 && term > 1e-300; ++j) { sum += term; term *= mu / (j + 1); }
      return sum * (double)nwin;
    };
    // a window with more rejections than RX fails over to the serial walker (never wrong, ~ms):
    // allowed with probability 1e-4 per step (~0.3 us of expected cost), not 1e-6
    const int RXr = tail(32) < 1e-4 ? 32 : tail(64) < 1e-4 ? 64 : 96;
    const int64_t ngrp = cdiv(nwin, CG);
    int* comp = reinterpret_cast<int*>(tables + a16(nwin * DWr));  // [ngroups][DW]
    int* tg = comp + ngrp * DWr;                                    // [ngroups]
    int* mid = tg + ngrp + 4;                                       // [nwin][DW]
    if (4 * n >= a16(4 * nwpos) + a16(16 * nwin) + 2 * a16(8 * nwin) + 64 + a16(nwin * DWr) +
                     4 * (ngrp * (DWr + 1) + 4 + nwin * DWr)) {  // room for the parallel walk
      // 4 launches to the bitmap: tables (+ scratch init + draw words), link (compose + chain +
      // rare serial fallback), emit_draws (+ hash insert), floyd_mark / tail shuffle
      RkInit ini{p.w.ticket, (16 + 8 * (nblk + 1)) / 4, p.w.bitmap, nwords, p.w.htab, 2 * p.w.H, p.w.ctl};
      const int64_t link_smem = 8 * ngrp + 2 * ngrp * DWr;
      const int stage_comp = link_smem <= RK_LINK_SMEM;
#define MC_RANDK_WALK(DWV, RXV)                                                                                        \
  {                                                                                                                   \
    const int ts = (DWV + RXV) * 32 * 4 + 1024 * HQ * 2 + (DWV + RXV) * 4;                                            \
    static std::atomic<uint64_t> cfg{0}, cfgl{0}; /* per device */                                                    \
    MC_API_CHECK(smem_optin(cfg, k_randk_tables<DWV, RXV>, ts));                                                      \
    note_launch(); k_randk_tables<DWV, RXV><<<(unsigned)nwin, 1024, ts, st>>>(p, p.w.list, nwpos, nwin, Lw, tables, ini); \
    const int ls = stage_comp ? (int)a16(link_smem) : 0;                                                              \
    MC_API_CHECK(smem_optin(cfgl, k_randk_link<DWV>, (int)a16(RK_LINK_SMEM)));                                         \
    note_launch(); k_randk_link<DWV><<<(unsigned)ngrp, 1024, ls, st>>>(p, p.w.list, nwpos, Lw, tables, nwin, comp, mid,  \
                                                                        tg, tin, ctl, p.w.ctl, stage_comp);           \
    note_launch(); k_randk_emit_draws<RXV><<<(unsigned)nwin, 1024, 0, st>>>(p, p.w.list, nwpos, tin, ctl);            \
  }
      if (DWr == 512 && RXr == 32) MC_RANDK_WALK(512, 32)
      else if (DWr == 512 && RXr == 64) MC_RANDK_WALK(512, 64)
      else if (DWr == 512) MC_RANDK_WALK(512, 96)
      else if (RXr == 32) MC_RANDK_WALK(1024, 32)
      else if (RXr == 64) MC_RANDK_WALK(1024, 64)
      else MC_RANDK_WALK(1024, 96)
#undef MC_RANDK_WALK
    } else {
      if (int rc = memsets()) return rc;
      note_launch(); k_randk_walk<<<1, 1024, 0, st>>>(p, p.w.list, 0);  // words generated on the fly
    }
    if (p.tail_shuffle) {
      note_launch(); k_randk_tail_shuffle<<<1, 1, 0, st>>>(p);
    } else {
      const unsigned gk = (unsigned)imax(1, imin(cdiv(k, 256), (int64_t)sm_count() * 8));
      note_launch(); k_randk_floyd_mark<<<gk, 256, 0, st>>>(p);
    }
  }
  const unsigned ge = (unsigned)cdiv(nwords, TB * RKW);
  note_launch();
#define MC_RK_EMIT(EF, MOM)                                                                      \
  if (vec) k_randk_emit<EF, MOM, true><<<rk_grid(k_randk_emit<EF, MOM, true>, ge), TB, 0, st>>>(p, ge); \
  else k_randk_emit<EF, MOM, false><<<rk_grid(k_randk_emit<EF, MOM, false>, ge), TB, 0, st>>>(p, ge);
  if (p.pro.r && p.pro.m) { MC_RK_EMIT(true, true) }
  else if (p.pro.r) { MC_RK_EMIT(true, false) }
  else if (p.pro.m) { MC_RK_EMIT(false, true) }
  else { MC_RK_EMIT(false, false) }
#undef MC_RK_EMIT
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int64_t decode_sparse_ws_bytes(int64_t n, int nranks) { return a16(4 * (int64_t)nranks * (cdiv(n, DT) + 1)); }

int decode_mean_sparse(const mc_spec* s, const mc_layout& L, const uint8_t* base, int64_t stride, int nranks, float* out,
                       const Ctx& c, void* ws, int64_t ws_bytes) {
  SD p{};
  p.base = base;
  p.stride = stride;
  p.nranks = nranks;
  p.n = L.n;
  p.ntiles = cdiv(L.n, DT);
  p.out = out;
  p.err = c.err;
  p.algo = (uint32_t)s->algorithm;
  // the per-(rank, tile) start table lives in the caller's workspace (no allocation here)
  const int64_t need = decode_sparse_ws_bytes(L.n, nranks);
  if (!ws || ws_bytes < need) {
    set_error("sparse decode workspace %lld < required %lld (mc_decode_workspace_bytes)", (long long)ws_bytes,
              (long long)need);
    return MC_EWORKSPACE;
  }
  p.starts = static_cast<uint32_t*>(ws);
  const int64_t maxcap = L.cap > 0 ? L.cap : L.n;
  dim3 g1((unsigned)imax(1, imin(cdiv(maxcap + 1, 256), (int64_t)sm_count() * 4)), (unsigned)nranks);
  note_launch(); k_sparse_starts<<<g1, 256, 0, c.stream>>>(p);
  note_launch(); k_sparse_tiles<<<(unsigned)p.ntiles, 256, 0, c.stream>>>(p);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

}  // namespace mc
