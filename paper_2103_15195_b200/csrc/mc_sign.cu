// mc_sign.cu — signsgd / signum (compressors.py:312-314; signum momentum :402-405).
//
// The single scaler is np.abs(x).mean() over the WHOLE group: numpy's float32 pairwise
// tree over n elements.  Every node at depth < D of that tree is internal (longer than
// 128) when P >> (D-1) >= 17 with P = n/8, and node offsets are multiples of 8, so:
//   pass 1  one warp per depth-D node (<= 512, or 1024 for groups > 117M elements): the
//           node's [offset, length) is
//           found by descending the numpy split rule from the root; the warp streams the
//           node once (momentum update, EF correction, sign bytes), stages |c32| in smem
//           and evaluates the node's bounded pairwise tree; the 8 warps of a CTA then
//           combine their 8 sibling nodes (a perfect subtree, 3 levels);
//   pass 2  one CTA combines the 2^(D-3) subtree sums as a perfect binary tree and
//           writes the scaler f32(f64(0 + P) / n);
//   pass 3  (error feedback only) r = c - (+-s).
#include <cstdlib>

#include "mc_internal.cuh"

namespace mc {
namespace {

constexpr int SW = 8;  // warps (nodes) per CTA in pass 1
constexpr int NODE_MAX = 2048;  // longest node the pass-1 kernels stage (16 chunks of 128)

struct SP {
  Prologue pro;
  int64_t n;
  float* partial;  // scratch: subtree sums
  int D;
  uint8_t* signs;  // payload bits
  float* scale;    // payload val[0]
  uint32_t* err;
  uint8_t* payload;
  mc_payload_header hdr;
};

// smem position of node element q: 8 pad floats per 32 so the (typically 4) leaves that the
// pairwise pass reads at once, ~n/4 apart, fall into disjoint bank octets; float4 aligned
__device__ __forceinline__ int spos(int q) { return pad32(q); }

// Streams the depth-D node [off, off + len) once; returns its pairwise sum (all lanes).
// Nodes start at multiples of 8 elements (so at sign-byte boundaries and 32-byte
// aligned) and hold <= 128*NCH elements: every lane issues all of its float4 loads of a
// group of 4 chunks before it touches any of them (one HBM round trip per group, not one
// per 32 elements), then writes sign bytes, the signum momentum, and |c32| to smem.
// MOM / EF are compile-time so the common signsgd node is a lean load/compare/store loop.
// Descends `levels` levels of the numpy split rule from the node [off, len): bit d of
// `path` = right child at the d-th level from the bottom.
__device__ __forceinline__ void split_descend(int path, int levels, int& off, int& len) {
  for (int d = levels - 1; d >= 0; --d) {
    const int m = (len >> 1) & ~7;  // n2 = n/2 - (n/2) % 8
    if ((path >> d) & 1) { off += m; len -= m; }
    else len = m;
  }
}

// `off`, `len`: the node's position (groups are < 2^31 elements; NODE_MAX check at launch)
template <int NCH, bool MOM, bool EF, bool VEC>
__device__ __forceinline__ float sign_node(const SP& p, int off, int len, float* a) {
  const int lane = threadIdx.x & 31;
  const int L = len;
  const float* g = p.pro.g + off;
  float* mo = MOM ? p.pro.m + off : nullptr;
  const double* r = EF ? p.pro.r + off : nullptr;
  float nanacc = 0.0f;  // x * 0 + acc stays 0 unless some x is inf / nan
#pragma unroll
  for (int c0 = 0; c0 < NCH; c0 += 4) {
    float xv[4][4], mv[4][4];
    double rv[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q0 = 128 * (c0 + i) + 4 * lane;
      if (VEC && q0 + 3 < L) {
        const float4 v = __ldcs(reinterpret_cast<const float4*>(g + q0));
        xv[i][0] = v.x; xv[i][1] = v.y; xv[i][2] = v.z; xv[i][3] = v.w;
        if (MOM) {
          const float4 u = *reinterpret_cast<const float4*>(mo + q0);
          mv[i][0] = u.x; mv[i][1] = u.y; mv[i][2] = u.z; mv[i][3] = u.w;
        }
        if (EF) {
          const double2 r0 = *reinterpret_cast<const double2*>(r + q0);
          const double2 r1 = *reinterpret_cast<const double2*>(r + q0 + 2);
          rv[i][0] = r0.x; rv[i][1] = r0.y; rv[i][2] = r1.x; rv[i][3] = r1.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool in = q0 + k < L;
          xv[i][k] = in ? g[q0 + k] : 0.0f;
          if (MOM) mv[i][k] = in ? mo[q0 + k] : 0.0f;
          if (EF) rv[i][k] = in ? r[q0 + k] : 0.0;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int q0 = 128 * (c0 + i) + 4 * lane;
      if (c0 + i > 0 && 128 * (c0 + i) >= L) break;  // warp-uniform: node ends before this chunk
      float c32[4];
      uint32_t nib = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = xv[i][k];
        nanacc = __fmaf_rn(x, 0.0f, nanacc);
        float w = x;
        if (MOM) {  // signum / momentum (compressors.py:402-405)
          w = p.pro.signum ? __fadd_rn(__fmul_rn(p.pro.beta, mv[i][k]), __fmul_rn(p.pro.omb, x))
                           : __fadd_rn(__fmul_rn(p.pro.beta, mv[i][k]), x);
          mv[i][k] = w;
        }
        c32[k] = EF ? __double2float_rn(__dadd_rn((double)w, rv[i][k])) : w;
        nib |= (uint32_t)(c32[k] >= 0.0f) << (3 - k);  // bit = x >= 0, MSB first
      }
      const bool full = q0 + 3 < L;
      if (!full) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (q0 + k >= L) nib &= ~(1u << (3 - k));  // np.packbits pads with zero bits
      }
      if (MOM) {
        if (VEC && full) {
          *reinterpret_cast<float4*>(mo + q0) = make_float4(mv[i][0], mv[i][1], mv[i][2], mv[i][3]);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (q0 + k < L) mo[q0 + k] = mv[i][k];
        }
      }
      // |c32| for the pairwise tree; lanes past the node end store zeros nobody reads
      *reinterpret_cast<float4*>(a + spos(q0)) = make_float4(fabsf(c32[0]), fabsf(c32[1]), fabsf(c32[2]), fabsf(c32[3]));
      // lanes 2j, 2j+1 hold the high / low nibble of sign byte j of this chunk
      uint32_t byte = nib << ((lane & 1) ? 0 : 4);
      byte |= __shfl_xor_sync(FULL, byte, 1);
      if (!(lane & 1) && q0 < L) p.signs[(off + q0) >> 3] = (uint8_t)byte;
    }
  }
  flag(p.err, nanacc != 0.0f, MC_ERR_NONFINITE);
  __syncwarp();
  // levels above the leaves (<= 128 elements): a split leaves children <= len/2 + 7.5, so
  // after d splits a node is <= L/2^d + 15; depth 3 holds up to L = 904, 4 up to 1808
  if (NCH <= 4 || L <= 904) return pairwise_pad32<3>(a, L);
  if (NCH <= 8 || L <= 1808) return pairwise_pad32<4>(a, L);
  return pairwise_pad32<5>(a, L);
}

template <int NCH, bool MOM, bool EF, bool VEC>
__global__ void __launch_bounds__(SW * 32) k_sign_nodes(SP p) {
  extern __shared__ __align__(16) float sm_dyn[];  // [SW][160 * NCH]
  float(*sm)[160 * NCH] = reinterpret_cast<float(*)[160 * NCH]>(sm_dyn);
  __shared__ float s_node[SW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int s_root[2];
  if (threadIdx.x == 0) {  // the CTA's 8 nodes share the top D-3 levels of the descent
    if (blockIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
    int off = 0, len = (int)p.n;
    split_descend((int)blockIdx.x, p.D - 3, off, len);
    s_root[0] = off;
    s_root[1] = len;
  }
  __syncthreads();
  int off = s_root[0], len = s_root[1];
  split_descend(warp, 3, off, len);
  const float s = sign_node<NCH, MOM, EF, VEC>(p, off, len, sm[warp]);
  if (lane == 0) s_node[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {  // nodes 8b .. 8b+7 form a perfect subtree (3 levels)
    const float l0 = __fadd_rn(s_node[0], s_node[1]), l1 = __fadd_rn(s_node[2], s_node[3]);
    const float l2 = __fadd_rn(s_node[4], s_node[5]), l3 = __fadd_rn(s_node[6], s_node[7]);
    p.partial[blockIdx.x] = __fadd_rn(__fadd_rn(l0, l1), __fadd_rn(l2, l3));
  }
}

// small trees (D < 3): one warp per node
template <bool MOM, bool EF>
__global__ void k_sign_nodes_small(SP p) {
  __shared__ __align__(16) float sm[160 * 16];
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  int off = 0, len = (int)p.n;
  split_descend((int)blockIdx.x, p.D, off, len);
  const float s = sign_node<16, MOM, EF, false>(p, off, len, sm);
  if (threadIdx.x == 0) p.partial[blockIdx.x] = s;
}

template <bool MOM, bool EF>
void launch_nodes(const SP& p, int64_t n, int64_t nodes, cudaStream_t st) {
  // node offsets are multiples of 8 elements: 16-byte aligned bases keep every node aligned
  const bool vec = (uintptr_t)p.pro.g % 16 == 0 && (!MOM || (uintptr_t)p.pro.m % 16 == 0) &&
                   (!EF || (uintptr_t)p.pro.r % 16 == 0);
  if (p.D >= 3) {
    // longest node at depth D is < (n >> D) + 8 (each split leaves the right child <= len/2 + 8)
    const dim3 grid((unsigned)(nodes / SW));
    const int64_t longest = (n >> p.D) + 16;
    constexpr int sm4 = SW * 160 * 4 * 4, sm8 = SW * 160 * 8 * 4, sm16 = SW * 160 * 16 * 4;
    if (longest <= 512) {
      if (vec) k_sign_nodes<4, MOM, EF, true><<<grid, SW * 32, sm4, st>>>(p);
      else k_sign_nodes<4, MOM, EF, false><<<grid, SW * 32, sm4, st>>>(p);
    } else if (longest <= 1024) {
      if (vec) k_sign_nodes<8, MOM, EF, true><<<grid, SW * 32, sm8, st>>>(p);
      else k_sign_nodes<8, MOM, EF, false><<<grid, SW * 32, sm8, st>>>(p);
    } else {
      static std::atomic<uint64_t> cfg_v{0}, cfg_s{0};
      smem_optin(cfg_v, k_sign_nodes<16, MOM, EF, true>, sm16);  // a failure surfaces at the launch check
      smem_optin(cfg_s, k_sign_nodes<16, MOM, EF, false>, sm16);
      if (vec) k_sign_nodes<16, MOM, EF, true><<<grid, SW * 32, sm16, st>>>(p);
      else k_sign_nodes<16, MOM, EF, false><<<grid, SW * 32, sm16, st>>>(p);
    }
  } else {
    k_sign_nodes_small<MOM, EF><<<(unsigned)nodes, 32, 0, st>>>(p);
  }
}

// perfect binary tree over m = 2^k values, in place with doubling strides:
// level l adds v[i + 2^l] into v[i] for i % 2^(l+1) == 0 (parent = left + right)
__global__ void k_sign_combine(SP p, int m) {
  extern __shared__ float v[];
  for (int i = threadIdx.x; i < m; i += blockDim.x) v[i] = p.partial[i];
  __syncthreads();
  for (int h = 1; h < m; h <<= 1) {
    for (int i = threadIdx.x * 2 * h; i < m; i += blockDim.x * 2 * h) v[i] = __fadd_rn(v[i], v[i + h]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *p.scale = np_mean(v[0], p.n);
}

__global__ void k_sign_ef(SP p) {
  const float s = *p.scale;
  const float ns = __fmul_rn(-1.0f, s);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p.n; e += (int64_t)gridDim.x * blockDim.x) {
    const float w = p.pro.m ? p.pro.m[e] : p.pro.g[e];  // momentum already advanced in pass 1
    const double c = __dadd_rn((double)w, p.pro.r[e]);
    const float c32 = __double2float_rn(c);
    p.pro.r[e] = __dsub_rn(c, (double)(c32 >= 0.0f ? s : ns));
  }
}

int sign_node_target() {
  static const int v = [] { const char* e = getenv("MC_SIGN_NODE"); return e ? atoi(e) : 880; }();
  return v;
}

int depth_for(int64_t n) {
  const int64_t P = n / 8;
  int D = 0;
  // every node at depth < D is split (length > 128); stop once nodes are <= ~800 elements
  while (D < 18 && (P >> D) >= 17 && (n >> D) > sign_node_target()) ++D;
  return D;
}

}  // namespace

int64_t signglobal_ws_bytes(const mc_spec*, int64_t n) { return a16(4 * ((1ll << depth_for(n)) + 64)) + 64; }

int encode_sign_global(const EncodeArgs& a) {
  SP p{};
  p.pro.g = a.g;
  p.pro.r = a.spec->error_feedback ? a.r : nullptr;
  p.pro.m = a.spec->has_momentum ? a.m : nullptr;
  p.pro.beta = a.spec->momentum;
  const float beta = a.spec->momentum;
  p.pro.omb = 1.0f - beta;
  p.pro.signum = a.spec->algorithm == MC_SIGNUM;
  p.n = a.n;
  p.partial = reinterpret_cast<float*>(a.ws);
  p.D = depth_for(a.n);
  p.signs = a.payload + a.L.off_bits;
  p.scale = reinterpret_cast<float*>(a.payload + a.L.off_val);
  p.err = a.ctx.err;
  p.payload = a.payload;
  p.hdr.algorithm = (uint32_t)a.spec->algorithm;
  p.hdr.original_len = (uint64_t)a.n;
  p.hdr.n_val = 1;
  p.hdr.n_bits = (uint32_t)a.L.n_bits;
  cudaStream_t st = a.ctx.stream;
  if ((a.n >> p.D) + 16 > NODE_MAX) {
    set_error("signsgd/signum group of %lld elements exceeds the supported 2^18 * 1000", (long long)a.n);
    return MC_EINVAL;
  }
  const int64_t nodes = 1ll << p.D;
  int m;
  note_launch();
  if (p.pro.m && p.pro.r) launch_nodes<true, true>(p, a.n, nodes, st);
  else if (p.pro.m) launch_nodes<true, false>(p, a.n, nodes, st);
  else if (p.pro.r) launch_nodes<false, true>(p, a.n, nodes, st);
  else launch_nodes<false, false>(p, a.n, nodes, st);
  m = (int)(p.D >= 3 ? nodes / SW : nodes);
  const int smem = 4 * m;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(k_sign_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
    set_error("signsgd combine needs %d bytes of shared memory", smem);
    return MC_ECUDA;
  }
  note_launch();
  k_sign_combine<<<1, 1024, smem, st>>>(p, m);
  if (p.pro.r) {
    const unsigned g = (unsigned)imax(1, imin(cdiv(a.n, 256), (int64_t)sm_count() * 8));
    note_launch();
    k_sign_ef<<<g, 256, 0, st>>>(p);
  }
  MC_LAUNCH_CHECK();
  return MC_OK;
}

}  // namespace mc
