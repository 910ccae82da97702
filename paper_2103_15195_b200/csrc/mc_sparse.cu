// mc_sparse.cu — sparsifiers: topk / dgc_lite (radix select), threshold (stream
// compaction), randk (numpy Generator.choice restated on device), and the fused
// sparse decode + rank-ordered mean.
//
// Reference: _compress compressors.py:272-289, randk :278-285, EF :409-413, decode
// :439-448, aggregate :519-532.  Tie contract for top-k: among
// equal |x| at the k-th boundary the LOWEST indices are kept.
#include "mc_internal.cuh"

namespace mc {
namespace {

constexpr int TB = 256;         // threads per compaction block
constexpr int ITEMS = 16;       // consecutive elements per thread
constexpr int TILE = TB * ITEMS;

// ------------------------------------------------------------------ workspace layout
struct SparseWS {
  uint32_t* keys;     // [n]  float bits of the corrected c32
  uint32_t* list;     // [n]  ordered candidate indices
  uint32_t* hist;     // [2048 + 2048 + 512]
  uint32_t* ctl;      // control words (see CTL_*)
  uint32_t* ticket;   // look-back ticket(s)
  uint64_t* status;   // look-back status [nblk]
  // randk
  uint32_t* draws;    // [k]   Floyd draws t_s
  uint32_t* htab;     // [2*H] hash (key, min step)
  uint32_t* bitmap;   // [ceil(n/32)]
  int64_t H;
};
enum { CTL_B1 = 0, CTL_KREM1, CTL_B2, CTL_KREM2, CTL_T, CTL_NEED, CTL_M, CTL_GT, CTL_COUNT, CTL_WORDS = 16 };

int64_t hash_size(int64_t k) {
  int64_t h = 1024;
  while (h < 4 * k) h <<= 1;
  return h;
}

SparseWS carve(uint8_t* w, int64_t n, int64_t k) {
  SparseWS s{};
  const int64_t nblk = cdiv(n, TILE) + 1;
  s.keys = reinterpret_cast<uint32_t*>(w); w += a16(4 * n);
  s.list = reinterpret_cast<uint32_t*>(w); w += a16(4 * n);
  s.hist = reinterpret_cast<uint32_t*>(w); w += a16(4 * (2048 + 2048 + 512));
  s.ctl = reinterpret_cast<uint32_t*>(w); w += a16(4 * CTL_WORDS);
  s.ticket = reinterpret_cast<uint32_t*>(w); w += 16;
  s.status = reinterpret_cast<uint64_t*>(w); w += a16(8 * nblk);
  s.H = hash_size(k);
  s.draws = reinterpret_cast<uint32_t*>(w); w += a16(4 * k);
  s.htab = reinterpret_cast<uint32_t*>(w); w += a16(8 * s.H);
  s.bitmap = reinterpret_cast<uint32_t*>(w); w += a16(4 * cdiv(n, 32));
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
struct TP {
  Prologue pro;
  int64_t n, k;
  SparseWS w;
  uint32_t* err;
  uint32_t* idx_out;
  float* val_out;
  uint8_t* payload;
  mc_payload_header hdr;
};

// pass 1: prologue (momentum, EF: r <- c in place), keys, 11-bit histogram of |c32|
__global__ void __launch_bounds__(256) k_topk_pass1(TP p) {
  __shared__ uint32_t h[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) h[i] = 0;
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  bool bad = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.n; e += (int64_t)gridDim.x * blockDim.x) {
    float c32;
    const double c = p.pro.load(e, c32, bad, true);
    if (p.pro.r) p.pro.r[e] = c;  // residual of unselected elements = c (compressors.py:412)
    const uint32_t bits = __float_as_uint(c32);
    p.w.keys[e] = bits;
    atomicAdd(&h[(bits & 0x7fffffffu) >> 20], 1u);
  }
  flag(p.err, bad, MC_ERR_NONFINITE);
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (h[i]) atomicAdd(&p.w.hist[i], h[i]);
}

// find the bin holding the k-th largest: scans nb bins from the top (one block of 1024)
__device__ void select_bin(const uint32_t* hist, int nb, uint32_t k, uint32_t* out_bin, uint32_t* out_krem) {
  __shared__ uint32_t s_w[32];
  // suffix sums: s_suf[i] = sum hist[i..nb)
  const int per = (nb + blockDim.x - 1) / blockDim.x;  // contiguous bins per thread, descending order
  const int t = threadIdx.x;
  // thread t owns bins [nb - (t+1)*per, nb - t*per)
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
  uint32_t run = s_w[warp] + incl - own;  // count of bins above my range
  for (int q = 0; q < per; ++q) {
    const int b = nb - t * per - 1 - q;
    if (b < 0) break;
    const uint32_t hb = hist[b];
    if (run < k && run + hb >= k) { *out_bin = (uint32_t)b; *out_krem = k - run; }
    run += hb;
  }
}

__global__ void k_topk_select1(TP p) {
  select_bin(p.w.hist, 2048, (uint32_t)p.k, &p.w.ctl[CTL_B1], &p.w.ctl[CTL_KREM1]);
}

// pass 2: ordered compaction of every element with bin1 >= B1 into the list; histogram
// of the next 11 key bits for the elements in bin B1.
__global__ void __launch_bounds__(TB) k_topk_pass2(TP p) {
  __shared__ uint32_t h2[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) h2[i] = 0;
  const int64_t bid = take_ticket(p.w.ticket);
  const uint32_t B1 = p.w.ctl[CTL_B1];
  const int64_t e0 = bid * TILE + (int64_t)threadIdx.x * ITEMS;
  uint32_t keep = 0;  // bitmask over my ITEMS
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const int64_t e = e0 + q;
    if (e < p.n) {
      const uint32_t key = p.w.keys[e] & 0x7fffffffu;
      const uint32_t b1 = key >> 20;
      if (b1 >= B1) keep |= 1u << q;
      if (b1 == B1) atomicAdd(&h2[(key >> 9) & 0x7ffu], 1u);
    }
  }
  uint64_t total;
  const uint64_t ex = block_exscan(__popc(keep), &total);
  const uint64_t pre = block_lookback(p.w.status, bid, total);
  uint64_t pos = pre + ex;
#pragma unroll
  for (int q = 0; q < ITEMS; ++q)
    if (keep & (1u << q)) p.w.list[pos++] = (uint32_t)(e0 + q);
  if (bid == (int64_t)gridDim.x - 1 && threadIdx.x == 0) p.w.ctl[CTL_M] = (uint32_t)(pre + total);
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    if (h2[i]) atomicAdd(&p.w.hist[2048 + i], h2[i]);
}

__global__ void k_topk_select2(TP p) {
  select_bin(p.w.hist + 2048, 2048, p.w.ctl[CTL_KREM1], &p.w.ctl[CTL_B2], &p.w.ctl[CTL_KREM2]);
}

// histogram of the low 9 key bits over list entries in (B1, B2)
__global__ void k_topk_hist3(TP p) {
  __shared__ uint32_t h3[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) h3[i] = 0;
  __syncthreads();
  const uint32_t M = p.w.ctl[CTL_M];
  const uint32_t hi = (p.w.ctl[CTL_B1] << 11) | p.w.ctl[CTL_B2];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = p.w.keys[p.w.list[i]] & 0x7fffffffu;
    if ((key >> 9) == hi) atomicAdd(&h3[key & 0x1ffu], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x)
    if (h3[i]) atomicAdd(&p.w.hist[4096 + i], h3[i]);
}

__global__ void k_topk_select3(TP p) {
  __shared__ uint32_t b3, need;
  select_bin(p.w.hist + 4096, 512, p.w.ctl[CTL_KREM2], &b3, &need);
  __syncthreads();
  if (threadIdx.x == 0) {
    p.w.ctl[CTL_T] = (p.w.ctl[CTL_B1] << 20) | (p.w.ctl[CTL_B2] << 9) | b3;
    p.w.ctl[CTL_NEED] = need;
  }
}

// final: ordered filter of the list: key > T, or key == T among the first `need` ties.
// Aggregate per block = (gt, ties) packed as 31|31 bits.
__global__ void __launch_bounds__(TB) k_topk_final(TP p) {
  const int64_t bid = take_ticket(p.w.ticket);
  const uint32_t M = p.w.ctl[CTL_M], T = p.w.ctl[CTL_T], need = p.w.ctl[CTL_NEED];
  if (bid * TILE >= (int64_t)M) return;  // no later block depends on an empty tail block
  const int64_t i0 = bid * TILE + (int64_t)threadIdx.x * ITEMS;
  uint32_t gt = 0, tie = 0;
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const int64_t i = i0 + q;
    if (i < M) {
      const uint32_t key = p.w.keys[p.w.list[i]] & 0x7fffffffu;
      gt |= (uint32_t)(key > T) << q;
      tie |= (uint32_t)(key == T) << q;
    }
  }
  const uint64_t mine = ((uint64_t)__popc(gt) << 31) | (uint64_t)__popc(tie);
  uint64_t total;
  const uint64_t ex = block_exscan(mine, &total);
  const uint64_t pre = block_lookback(p.w.status, bid, total);
  const uint64_t before = pre + ex;
  uint64_t gt_before = before >> 31, tie_before = before & 0x7fffffffull;
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const bool is_gt = gt & (1u << q), is_tie = tie & (1u << q);
    if (is_gt || (is_tie && tie_before < need)) {
      const uint64_t slot = gt_before + (tie_before < need ? tie_before : need);
      const uint32_t e = p.w.list[i0 + q];
      const float c32 = __uint_as_float(p.w.keys[e]);
      p.idx_out[slot] = e;
      p.val_out[slot] = c32;
      if (p.pro.r) p.pro.r[e] = __dsub_rn(p.pro.r[e], (double)c32);  // r = c - decode  (:412)
    }
    gt_before += is_gt;
    tie_before += is_tie;
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
  uint8_t* payload;
  mc_payload_header hdr;
};

__global__ void __launch_bounds__(TB) k_threshold(ThP p) {
  const int64_t bid = take_ticket(p.ticket);
  const int64_t e0 = bid * TILE + (int64_t)threadIdx.x * ITEMS;
  float v[ITEMS];
  uint32_t keep = 0;
  bool bad = false;
#pragma unroll
  for (int q = 0; q < ITEMS; ++q) {
    const int64_t e = e0 + q;
    v[q] = 0.0f;
    if (e < p.n) {
      float c32;
      const double c = p.pro.load(e, c32, bad, true);
      v[q] = c32;
      const bool sel = fabsf(c32) >= p.tau;  // |x| >= f32(tau)  (compressors.py:288)
      keep |= (uint32_t)sel << q;
      if (p.pro.r) p.pro.r[e] = sel ? __dsub_rn(c, (double)c32) : c;
    }
  }
  flag(p.err, bad, MC_ERR_NONFINITE);
  uint64_t total;
  const uint64_t ex = block_exscan(__popc(keep), &total);
  const uint64_t pre = block_lookback(p.status, bid, total);
  uint64_t pos = pre + ex;
#pragma unroll
  for (int q = 0; q < ITEMS; ++q)
    if (keep & (1u << q)) {
      p.idx_out[pos] = (uint32_t)(e0 + q);
      p.val_out[pos] = v[q];
      ++pos;
    }
  if (bid == (int64_t)gridDim.x - 1 && threadIdx.x == 0) {
    mc_payload_header h = p.hdr;
    h.n_idx = h.n_val = (uint32_t)(pre + total);
    *reinterpret_cast<mc_payload_header*>(p.payload) = h;
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
  int unbiased;
  int tail_shuffle;  // numpy's tail-shuffle branch (k > n//50 and n > 10000)
  uint8_t* payload;
  mc_payload_header hdr;
};

__device__ __forceinline__ uint32_t draw32(const Philox& ph, uint64_t pos) {
  uint64_t w[4];
  ph.block(pos >> 3, w);
  const uint64_t x = w[(pos >> 1) & 3];
  return (pos & 1) ? (uint32_t)(x >> 32) : (uint32_t)x;
}

// One warp walks the draw stream: step s consumes draws until Lemire accepts for
// range j_s (Floyd: j_s = n-k+s ascending; tail shuffle: j_s = n-1-s descending).
__global__ void k_randk_walk(RP p) {
  const int lane = threadIdx.x;
  const Philox ph{p.k0, p.k1};
  uint64_t s = 0, pos = 0;
  while (s < (uint64_t)p.k) {
    const uint64_t my = s + lane;
    bool rej = false;
    uint32_t val = 0;
    if (my < (uint64_t)p.k) {
      const uint64_t j = p.tail_shuffle ? (uint64_t)(p.n - 1) - my : (uint64_t)(p.n - p.k) + my;
      if (j == 0) {
        val = 0;  // random_bounded_uint64(rng=0) returns without drawing
      } else {
        const uint64_t excl = j + 1;
        const uint64_t m = (uint64_t)draw32(ph, pos + lane) * excl;
        const uint32_t left = (uint32_t)m;
        if (left < excl) {
          const uint32_t thr = (uint32_t)((0x100000000ull - excl) % excl);
          rej = left < thr;
        }
        val = (uint32_t)(m >> 32);
      }
    }
    // j == 0 consumes no draw: only possible for the very first Floyd step with k == n,
    // which the host routes to the full selection path.
    const unsigned rm = __ballot_sync(FULL, rej);
    const int f = rm ? __ffs(rm) - 1 : 32;
    if (lane < f && my < (uint64_t)p.k) p.w.draws[my] = val;
    s += f;
    pos += f + (rm ? 1 : 0);
  }
}

__device__ __forceinline__ uint32_t hslot(uint32_t key, int64_t H) { return (key * 0x9E3779B1u) & (uint32_t)(H - 1); }

__global__ void k_randk_insert(RP p) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < p.k; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = p.w.draws[s];
    uint32_t h = hslot(key, p.w.H);
    while (true) {
      const uint32_t prev = atomicCAS(&p.w.htab[2 * h], 0xffffffffu, key);
      if (prev == 0xffffffffu || prev == key) { atomicMin(&p.w.htab[2 * h + 1], (uint32_t)s); break; }
      h = (h + 1) & (uint32_t)(p.w.H - 1);
    }
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

// ordered compaction of the bitmap -> ascending indices; gather values; EF fix-up
__global__ void __launch_bounds__(TB) k_randk_emit(RP p) {
  const int64_t bid = take_ticket(p.w.ticket);
  const int64_t nw = cdiv(p.n, 32);
  const int64_t w0 = bid * TB * 4 + (int64_t)threadIdx.x * 4;  // 4 words (128 elements) per thread
  uint32_t words[4];
  uint32_t cnt = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    words[q] = (w0 + q < nw) ? p.w.bitmap[w0 + q] : 0u;
    cnt += __popc(words[q]);
  }
  uint64_t total;
  const uint64_t ex = block_exscan(cnt, &total);
  const uint64_t pre = block_lookback(p.w.status, bid, total);
  uint64_t pos = pre + ex;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t m = words[q];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int64_t e = (w0 + q) * 32 + b;
      float c32;
      bool bad = false;
      double c;
      if (p.pro.r) {
        c = p.pro.r[e];  // pass 1 stored r <- c
        c32 = __double2float_rn(c);
      } else {
        c32 = p.pro.m ? p.pro.m[e] : p.pro.g[e];
        c = (double)c32;
      }
      (void)bad;
      const float v = p.unbiased ? __fmul_rn(c32, p.scale) : c32;
      p.idx_out[pos] = (uint32_t)e;
      p.val_out[pos] = v;
      if (p.pro.r) p.pro.r[e] = __dsub_rn(c, (double)v);
      ++pos;
    }
  }
}

// prologue pass for randk (momentum/EF state update, non-finite check; no keys needed)
__global__ void k_sparse_prologue(Prologue pro, int64_t n, uint32_t* err, uint8_t* payload, mc_payload_header hdr) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(payload) = hdr;
  bool bad = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    float c32;
    const double c = pro.load(e, c32, bad, true);
    if (pro.r) pro.r[e] = c;
  }
  flag(err, bad, MC_ERR_NONFINITE);
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
constexpr int DT = 4096;  // output tile (elements)

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

__global__ void __launch_bounds__(512) k_sparse_tiles(SD p) {
  __shared__ float acc[DT];
  const int64_t t = blockIdx.x;
  const int64_t t0 = t * DT;
  for (int i = threadIdx.x; i < DT; i += blockDim.x) acc[i] = 0.0f;
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
  const int64_t lim = imin(DT, p.n - t0);
  for (int i = threadIdx.x; i < lim; i += blockDim.x) p.out[t0 + i] = __fdiv_rn(acc[i], fn);
}

}  // namespace

int64_t sparse_ws_bytes(const mc_spec* s, int64_t n) {
  const int64_t k = s->algorithm == MC_THRESHOLD ? 1 : top_k_count(s->sparsity, n);
  const int64_t nblk = cdiv(n, TILE) + 1;
  return a16(4 * n) * 2 + a16(4 * (2048 + 2048 + 512)) + a16(4 * CTL_WORDS) + 16 + a16(8 * nblk) + a16(4 * k) +
         a16(8 * hash_size(k)) + a16(4 * cdiv(n, 32)) + 64;
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

int encode_topk(const EncodeArgs& a) {
  const int64_t n = a.n, k = top_k_count(a.spec->sparsity, n);
  TP p{};
  p.pro = make_prologue(a);
  p.n = n;
  p.k = k;
  p.w = carve(a.ws, n, k);
  p.err = a.ctx.err;
  p.idx_out = reinterpret_cast<uint32_t*>(a.payload + a.L.off_idx);
  p.val_out = reinterpret_cast<float*>(a.payload + a.L.off_val);
  p.payload = a.payload;
  p.hdr.algorithm = (uint32_t)a.spec->algorithm;
  p.hdr.original_len = (uint64_t)n;
  p.hdr.n_idx = p.hdr.n_val = p.hdr.cap = (uint32_t)k;
  cudaStream_t st = a.ctx.stream;
  const int64_t nblk = cdiv(n, TILE);
  // zero histograms + ctl + ticket + status in one memset (contiguous in the carve)
  const size_t zbytes = (size_t)((uint8_t*)p.w.status - (uint8_t*)p.w.hist) + 8 * (nblk + 1);
  if (cudaMemsetAsync(p.w.hist, 0, zbytes, st) != cudaSuccess) return MC_ECUDA;
  const unsigned g1 = (unsigned)imax(1, imin(cdiv(n, 256), (int64_t)sm_count() * 4));
  note_launch(); k_topk_pass1<<<g1, 256, 0, st>>>(p);
  note_launch(); k_topk_select1<<<1, 1024, 0, st>>>(p);
  note_launch(); k_topk_pass2<<<(unsigned)nblk, TB, 0, st>>>(p);
  note_launch(); k_topk_select2<<<1, 1024, 0, st>>>(p);
  note_launch(); k_topk_hist3<<<(unsigned)sm_count(), 256, 0, st>>>(p);
  note_launch(); k_topk_select3<<<1, 1024, 0, st>>>(p);
  // reset ticket + status for the final look-back pass (list length <= n)
  if (cudaMemsetAsync(p.w.ticket, 0, 16 + 8 * (nblk + 1), st) != cudaSuccess) return MC_ECUDA;
  note_launch(); k_topk_final<<<(unsigned)nblk, TB, 0, st>>>(p);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int encode_threshold(const EncodeArgs& a) {
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
  const int64_t nblk = cdiv(n, TILE);
  cudaStream_t st = a.ctx.stream;
  if (cudaMemsetAsync(w.ticket, 0, 16 + 8 * (nblk + 1), st) != cudaSuccess) return MC_ECUDA;
  note_launch(); k_threshold<<<(unsigned)nblk, TB, 0, st>>>(p);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int encode_randk(const EncodeArgs& a) {
  const int64_t n = a.n, k = top_k_count(a.spec->sparsity, n);
  RP p{};
  p.pro = make_prologue(a);
  p.n = n;
  p.k = k;
  p.k0 = a.k0;
  p.k1 = a.k1;
  p.w = carve(a.ws, n, k);
  p.err = a.ctx.err;
  p.idx_out = reinterpret_cast<uint32_t*>(a.payload + a.L.off_idx);
  p.val_out = reinterpret_cast<float*>(a.payload + a.L.off_val);
  p.unbiased = a.spec->unbiased_scaling;
  p.scale = (float)((double)n / (double)k);  // np.float32(n / k)  (compressors.py:284)
  p.tail_shuffle = (n > 10000 && k > n / 50) ? 1 : 0;
  p.payload = a.payload;
  p.hdr.algorithm = MC_RANDK;
  p.hdr.flags = p.unbiased ? 1u : 0u;
  p.hdr.original_len = (uint64_t)n;
  p.hdr.n_idx = p.hdr.n_val = p.hdr.cap = (uint32_t)k;
  cudaStream_t st = a.ctx.stream;
  const int64_t nwords = cdiv(n, 32);
  const int64_t nblk = cdiv(nwords, TB * 4) + 1;
  if (cudaMemsetAsync(p.w.ticket, 0, 16 + 8 * (nblk + 1), st) != cudaSuccess) return MC_ECUDA;
  if (cudaMemsetAsync(p.w.bitmap, 0, 4 * nwords, st) != cudaSuccess) return MC_ECUDA;
  if (cudaMemsetAsync(p.w.htab, 0xff, 8 * p.w.H, st) != cudaSuccess) return MC_ECUDA;
  const unsigned g1 = (unsigned)imax(1, imin(cdiv(n, 256), (int64_t)sm_count() * 4));
  note_launch(); k_sparse_prologue<<<g1, 256, 0, st>>>(p.pro, n, p.err, p.payload, p.hdr);
  if (k == n) {
    note_launch(); k_bitmap_all<<<(unsigned)imax(1, imin(cdiv(nwords, 256), 1024)), 256, 0, st>>>(p);
  } else {
    note_launch(); k_randk_walk<<<1, 32, 0, st>>>(p);
    if (p.tail_shuffle) {
      note_launch(); k_randk_tail_shuffle<<<1, 1, 0, st>>>(p);
    } else {
      const unsigned gk = (unsigned)imax(1, imin(cdiv(k, 256), (int64_t)sm_count() * 8));
      note_launch(); k_randk_insert<<<gk, 256, 0, st>>>(p);
      note_launch(); k_randk_floyd_mark<<<gk, 256, 0, st>>>(p);
    }
  }
  note_launch(); k_randk_emit<<<(unsigned)cdiv(nwords, TB * 4), TB, 0, st>>>(p);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

int decode_mean_sparse(const mc_spec* s, const mc_layout& L, const uint8_t* base, int64_t stride, int nranks, float* out,
                       const Ctx& c) {
  SD p{};
  p.base = base;
  p.stride = stride;
  p.nranks = nranks;
  p.n = L.n;
  p.ntiles = cdiv(L.n, DT);
  p.out = out;
  p.err = c.err;
  p.algo = (uint32_t)s->algorithm;
  // the tile-start table lives in a stream-ordered scratch allocation
  const size_t bytes = 4 * (size_t)nranks * (size_t)(p.ntiles + 1);
  void* scratch = nullptr;
  if (cudaMallocAsync(&scratch, bytes, c.stream) != cudaSuccess) {
    set_error("cudaMallocAsync(%zu) failed", bytes);
    return MC_ECUDA;
  }
  p.starts = static_cast<uint32_t*>(scratch);
  const int64_t maxcap = L.cap > 0 ? L.cap : L.n;
  dim3 g1((unsigned)imax(1, imin(cdiv(maxcap + 1, 256), (int64_t)sm_count() * 4)), (unsigned)nranks);
  note_launch(); k_sparse_starts<<<g1, 256, 0, c.stream>>>(p);
  note_launch(); k_sparse_tiles<<<(unsigned)p.ntiles, 512, 0, c.stream>>>(p);
  cudaFreeAsync(scratch, c.stream);
  MC_LAUNCH_CHECK();
  return MC_OK;
}

}  // namespace mc
