// mc_sign.cu — signsgd / signum (compressors.py:312-314; signum momentum :402-405).
//
// The single scaler is np.abs(x).mean() over the WHOLE group: numpy's float32 pairwise
// tree over n elements.  Every node at depth < D of that tree is internal (longer than
// 128) when P >> (D-1) >= 17 with P = n/8, and node offsets are multiples of 8, so:
//   pass 1  one warp per depth-D node (<= ~800 elements): the node's [offset, length) is
//           found by descending the numpy split rule from the root; the warp streams the
//           node once (momentum update, EF correction, sign bytes), stages |c32| in smem
//           and evaluates the node's bounded pairwise tree; the 8 warps of a CTA then
//           combine their 8 sibling nodes (a perfect subtree, 3 levels);
//   pass 2  one CTA combines the 2^(D-3) subtree sums as a perfect binary tree and
//           writes the scaler f32(f64(0 + P) / n);
//   pass 3  (error feedback only) r = c - (+-s).
#include "mc_internal.cuh"

namespace mc {
namespace {

constexpr int SW = 8;  // warps (nodes) per CTA in pass 1
constexpr int NODE_MAX = 1024;

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

// Streams node `node` (depth D) once; returns the node's pairwise sum (all lanes).
__device__ __forceinline__ float sign_node(const SP& p, int64_t node, float* a) {
  const int lane = threadIdx.x & 31;
  int64_t off = 0, len = p.n;
  for (int d = p.D - 1; d >= 0; --d) {  // bit d of the node index = right child at that level
    int64_t m = len / 2;
    m -= m % 8;
    if ((node >> d) & 1) { off += m; len -= m; }
    else len = m;
  }
  bool bad = false;
  for (int64_t q0 = 0; q0 < len; q0 += 32) {
    const int64_t q = q0 + lane;
    float c32 = 0.0f;
    if (q < len) {
      p.pro.load(off + q, c32, bad, true);
      a[q] = fabsf(c32);
    }
    const unsigned m = __ballot_sync(FULL, q < len && c32 >= 0.0f);  // bit = x >= 0
    if (lane < 4 && q0 + 8 * lane < len)  // elements 8*lane .. +7 of this chunk, MSB first
      p.signs[(off + q0) / 8 + lane] = (uint8_t)((__brev(m) >> (24 - 8 * lane)) & 0xffu);
  }
  flag(p.err, bad, MC_ERR_NONFINITE);
  __syncwarp();
  return warp_pairwise_small<4>([&](int q) { return a[q]; }, (int)len);
}

__global__ void __launch_bounds__(SW * 32) k_sign_nodes(SP p) {
  __shared__ __align__(16) float sm[SW][NODE_MAX];
  __shared__ float s_node[SW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  const float s = sign_node(p, (int64_t)blockIdx.x * SW + warp, sm[warp]);
  if (lane == 0) s_node[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {  // nodes 8b .. 8b+7 form a perfect subtree (3 levels)
    const float l0 = __fadd_rn(s_node[0], s_node[1]), l1 = __fadd_rn(s_node[2], s_node[3]);
    const float l2 = __fadd_rn(s_node[4], s_node[5]), l3 = __fadd_rn(s_node[6], s_node[7]);
    p.partial[blockIdx.x] = __fadd_rn(__fadd_rn(l0, l1), __fadd_rn(l2, l3));
  }
}

// small trees (D < 3): one warp per node
__global__ void k_sign_nodes_small(SP p) {
  __shared__ __align__(16) float sm[NODE_MAX];
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  const float s = sign_node(p, blockIdx.x, sm);
  if (threadIdx.x == 0) p.partial[blockIdx.x] = s;
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

int depth_for(int64_t n) {
  const int64_t P = n / 8;
  int D = 0;
  // every node at depth < D is split (length > 128); stop once nodes are <= ~800 elements
  while (D < 18 && (P >> D) >= 17 && (n >> D) > 768) ++D;
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
  if (p.D >= 3) {
    k_sign_nodes<<<(unsigned)(nodes / SW), SW * 32, 0, st>>>(p);
    m = (int)(nodes / SW);
  } else {
    k_sign_nodes_small<<<(unsigned)nodes, 32, 0, st>>>(p);
    m = (int)nodes;
  }
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
