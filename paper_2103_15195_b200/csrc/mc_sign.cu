// mc_sign.cu — signsgd / signum (compressors.py:312-314; signum momentum :402-405).
//
// The single scaler is np.abs(x).mean() over the WHOLE group: numpy's float32
// pairwise tree over n elements.  All nodes at depth < D of that tree are internal
// (their length exceeds 128) when P >> (D-1) >= 17 with P = n/8, so
//   pass 1  writes |c32| to scratch + the sign words (warp ballots), updates momentum;
//   pass 2  one warp per depth-D node: the node's [offset, length) is found by
//           descending from the root with the numpy split rule, then the warp
//           evaluates the pairwise recursion of that node;
//   pass 3  one block combines the 2^D node sums as a perfect binary tree and
//           writes the scaler (f32(f64(0 + P) / n));
//   pass 4  (error feedback only) r = c - (+-s).
#include "mc_internal.cuh"

namespace mc {
namespace {

struct SP {
  Prologue pro;
  int64_t n;
  float* absx;       // scratch [n]
  float* nodes;      // scratch [2^D]
  int D;
  uint32_t* signs;   // payload bits (u32 words)
  float* scale;      // payload val[0]
  uint32_t* err;
  uint8_t* payload;
  mc_payload_header hdr;
};

__global__ void k_sign_pass1(SP p) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<mc_payload_header*>(p.payload) = p.hdr;
  bool bad = false;
  const int lane = threadIdx.x & 31;
  const int64_t nwords = cdiv(p.n, 32);
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords; w += warps) {
    const int64_t e = w * 32 + lane;
    float c32 = 0.0f;
    if (e < p.n) {
      p.pro.load(e, c32, bad, true);
      p.absx[e] = fabsf(c32);
    }
    const unsigned m = __ballot_sync(FULL, e < p.n && c32 >= 0.0f);
    if (lane == 0) p.signs[w] = __byte_perm(__brev(m), 0, 0x0123);
  }
  flag(p.err, bad, MC_ERR_NONFINITE);
}

__global__ void k_sign_nodes(SP p) {
  const int64_t node = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (node >= (1ll << p.D)) return;
  int64_t off = 0, len = p.n;
  for (int d = p.D - 1; d >= 0; --d) {  // descend: bit d of node = go right at that level
    int64_t m = len / 2;
    m -= m % 8;
    if ((node >> d) & 1) { off += m; len -= m; }
    else len = m;
  }
  const float* a = p.absx + off;
  const float s = warp_pairwise([&](int64_t q) { return a[q]; }, len);
  if ((threadIdx.x & 31) == 0) p.nodes[node] = s;
}

__global__ void k_sign_combine(SP p) {
  __shared__ float v[4096];
  const int N = 1 << p.D;
  for (int i = threadIdx.x; i < N; i += blockDim.x) v[i] = p.nodes[i];
  __syncthreads();
  for (int w = N >> 1; w >= 1; w >>= 1) {  // level by level: parent = left + right
    float t[4];
    int cnt = 0;
    for (int i = threadIdx.x; i < w; i += blockDim.x) t[cnt++] = __fadd_rn(v[2 * i], v[2 * i + 1]);
    __syncthreads();
    cnt = 0;
    for (int i = threadIdx.x; i < w; i += blockDim.x) v[i] = t[cnt++];
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
  while (D < 12 && (P >> D) >= 17) ++D;  // every node at depth < D has length > 128
  return D;
}

}  // namespace

int64_t signglobal_ws_bytes(const mc_spec*, int64_t n) { return a16(4 * n) + a16(4 * 4096) + 64; }

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
  p.absx = reinterpret_cast<float*>(a.ws);
  p.nodes = reinterpret_cast<float*>(a.ws + a16(4 * a.n));
  p.D = depth_for(a.n);
  p.signs = reinterpret_cast<uint32_t*>(a.payload + a.L.off_bits);
  p.scale = reinterpret_cast<float*>(a.payload + a.L.off_val);
  p.err = a.ctx.err;
  p.payload = a.payload;
  p.hdr.algorithm = (uint32_t)a.spec->algorithm;
  p.hdr.original_len = (uint64_t)a.n;
  p.hdr.n_val = 1;
  p.hdr.n_bits = (uint32_t)a.L.n_bits;
  cudaStream_t st = a.ctx.stream;
  // pass 1 reads the un-advanced momentum and advances it: the EF pass then reads m'.
  const int64_t warps = cdiv(a.n, 32);
  const unsigned g1 = (unsigned)imax(1, imin(cdiv(warps * 32, 256), (int64_t)sm_count() * 8));
  note_launch(); k_sign_pass1<<<g1, 256, 0, st>>>(p);
  const int64_t nodes = 1ll << p.D;
  note_launch(); k_sign_nodes<<<(unsigned)cdiv(nodes * 32, 256), 256, 0, st>>>(p);
  note_launch(); k_sign_combine<<<1, 1024, 0, st>>>(p);
  if (p.pro.r) {
    const unsigned g = (unsigned)imax(1, imin(cdiv(a.n, 256), (int64_t)sm_count() * 8));
    note_launch(); k_sign_ef<<<g, 256, 0, st>>>(p);
  }
  MC_LAUNCH_CHECK();
  return MC_OK;
}

}  // namespace mc
