// mc_pipe.cu — native host-buffer sync for one rank (the e2e path a trainer on host
// memory takes): pinned host gradients -> device, fused encode + single-rank aggregate,
// averaged gradients -> host, all enqueued from C++ on three caller streams so PCIe runs
// full duplex and the CPU issues each chunk in microseconds (no interpreter per chunk).
//
//   H2D stream   chunk c of this call waits for the previous call's read-out of the same
//                device chunk (event), then copies host_in -> dev
//   encode       chunkable codecs (identity, fp16, efsignsgd, onebit, int8): per chunk,
//                mc_encode_range with out = dev (in place); others: the whole group with
//                mc_encode_decode after its last H2D chunk
//   D2H stream   per chunk after its encode: dev -> host_out, event kept for the next call
//
// Reference: the trainer's per-step sync of one worker's host gradient
// (trainer.py:360-395 with one worker), compressors.py encode/aggregate.
#include <unordered_map>
#include <vector>

#include "mc_internal.cuh"

struct mc_pipe {
  std::unordered_map<uintptr_t, cudaEvent_t> last_out;  // device chunk address -> its last D2H
  std::vector<cudaEvent_t> pool;                        // free events
  std::vector<cudaEvent_t> live;                        // events owned by this call (recycled next call)
  cudaEvent_t enc_done = nullptr, out_done = nullptr;
  int device = -1;
};

namespace {

cudaError_t take_event(mc_pipe* p, cudaEvent_t* ev) {
  if (!p->pool.empty()) {
    *ev = p->pool.back();
    p->pool.pop_back();
    return cudaSuccess;
  }
  return cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
}

bool chunkable(int algo) {
  return algo == MC_IDENTITY || algo == MC_FP16 || algo == MC_EFSIGNSGD || algo == MC_ONEBIT || algo == MC_INT8;
}

int64_t gcd64(int64_t a, int64_t b) { return b ? gcd64(b, a % b) : a; }

}  // namespace

using namespace mc;

extern "C" {

int mc_pipe_create(mc_pipe** out) {
  if (!out) { set_error("null output"); return MC_EINVAL; }
  mc_pipe* p = new (std::nothrow) mc_pipe();
  if (!p) { set_error("out of host memory"); return MC_EINVAL; }
  cudaGetDevice(&p->device);
  *out = p;
  return MC_OK;
}

void mc_pipe_destroy(mc_pipe* p) {
  if (!p) return;
  for (auto& kv : p->last_out) cudaEventDestroy(kv.second);
  for (cudaEvent_t e : p->pool) cudaEventDestroy(e);
  for (cudaEvent_t e : p->live) cudaEventDestroy(e);
  delete p;
}

int mc_pipe_group(mc_pipe* p, const mc_spec* s, const float* host_in, float* host_out, float* dev, int64_t n,
                  int64_t chunk, double* residual, float* momentum, uint64_t key_lo, uint64_t key_hi, void* payload,
                  void* workspace, int64_t workspace_bytes, uint32_t* err_flags, void* s_h2d, void* s_enc,
                  void* s_d2h) {
  if (!p || !s || !host_in || !host_out || !dev || n < 1 || chunk < 1) {
    set_error("bad mc_pipe_group arguments");
    return MC_EINVAL;
  }
  cudaStream_t sh = static_cast<cudaStream_t>(s_h2d), se = static_cast<cudaStream_t>(s_enc),
               sd = static_cast<cudaStream_t>(s_d2h);
  const bool per_chunk = chunkable(s->algorithm);
  if (per_chunk) {  // chunks on bucket and sign-word boundaries
    const int64_t align = (s->algorithm == MC_IDENTITY || s->algorithm == MC_FP16)
                              ? 32 : s->bucket_size / gcd64(s->bucket_size, 32) * 32;
    chunk = chunk < align ? align : chunk / align * align;
  } else {
    chunk = (chunk + 31) / 32 * 32;
  }
  // chunk schedule: tapered at both ends (chunk/8, /4, /2 ... /2, /4, /8) so the pipeline
  // fill (first H2D alone) and drain (last D2H alone) cost a small chunk, not a full one
  int64_t align = 32;
  if (per_chunk && s->algorithm != MC_IDENTITY && s->algorithm != MC_FP16)
    align = s->bucket_size / gcd64(s->bucket_size, 32) * 32;
  std::vector<int64_t> sizes;
  {
    const int64_t q = chunk / 8 / align * align;
    int64_t head[3] = {q, 2 * q, 4 * q};
    int64_t used = 0;
    if (q >= align && n >= 4 * chunk) {
      for (int64_t h : head) { sizes.push_back(h); used += h; }
      used += 7 * q;  // the mirrored tail
    }
    // middle chunks stay aligned; the group's unaligned remainder rides on its last chunk
    int64_t mid = (n - used) / align * align;
    const int64_t rem = n - used - mid;
    while (mid > 0) { const int64_t c = imin(chunk, mid); sizes.push_back(c); mid -= c; }
    if (used) for (int i = 2; i >= 0; --i) sizes.push_back(head[i]);
    if (rem) {
      if (sizes.empty()) sizes.push_back(rem);
      else sizes.back() += rem;
    }
  }
  const int64_t nch = (int64_t)sizes.size();
  cudaEvent_t ev_in = nullptr;
  int64_t b = 0;
  for (int64_t c = 0; c < nch; b += sizes[c], ++c) {
    const int64_t cnt = sizes[c];
    const uintptr_t key = reinterpret_cast<uintptr_t>(dev + b);
    auto it = p->last_out.find(key);
    if (it != p->last_out.end()) MC_API_CHECK(cudaStreamWaitEvent(sh, it->second, 0));
    MC_API_CHECK(cudaMemcpyAsync(dev + b, host_in + b, 4 * cnt, cudaMemcpyHostToDevice, sh));
    if (!per_chunk && c + 1 < nch) continue;
    MC_API_CHECK(take_event(p, &ev_in));
    p->live.push_back(ev_in);
    MC_API_CHECK(cudaEventRecord(ev_in, sh));
    if (per_chunk) {
      MC_API_CHECK(cudaStreamWaitEvent(se, ev_in, 0));
      const int rc = mc_encode_range(s, dev, n, b, cnt, residual, momentum, key_lo, key_hi, payload, workspace,
                                     workspace_bytes, dev, err_flags, se);
      if (rc != MC_OK) return rc;
      cudaEvent_t ev_c;
      MC_API_CHECK(take_event(p, &ev_c));
      p->live.push_back(ev_c);
      MC_API_CHECK(cudaEventRecord(ev_c, se));
      MC_API_CHECK(cudaStreamWaitEvent(sd, ev_c, 0));
      MC_API_CHECK(cudaMemcpyAsync(host_out + b, dev + b, 4 * cnt, cudaMemcpyDeviceToHost, sd));
      cudaEvent_t ev_o;
      MC_API_CHECK(take_event(p, &ev_o));
      MC_API_CHECK(cudaEventRecord(ev_o, sd));
      auto jt = p->last_out.find(key);
      if (jt != p->last_out.end()) { p->live.push_back(jt->second); jt->second = ev_o; }
      else p->last_out.emplace(key, ev_o);
    }
  }
  if (!per_chunk) {  // whole-group encode after the last H2D chunk, then chunked read-out
    MC_API_CHECK(cudaStreamWaitEvent(se, ev_in, 0));
    const int rc = mc_encode_decode(s, dev, n, residual, momentum, key_lo, key_hi, payload, workspace,
                                    workspace_bytes, dev, err_flags, se);
    if (rc != MC_OK) return rc;
    cudaEvent_t ev_c;
    MC_API_CHECK(take_event(p, &ev_c));
    p->live.push_back(ev_c);
    MC_API_CHECK(cudaEventRecord(ev_c, se));
    MC_API_CHECK(cudaStreamWaitEvent(sd, ev_c, 0));
    int64_t b = 0;
    for (int64_t c = 0; c < nch; b += sizes[c], ++c) {
      const int64_t cnt = sizes[c];
      const uintptr_t key = reinterpret_cast<uintptr_t>(dev + b);
      MC_API_CHECK(cudaMemcpyAsync(host_out + b, dev + b, 4 * cnt, cudaMemcpyDeviceToHost, sd));
      cudaEvent_t ev_o;
      MC_API_CHECK(take_event(p, &ev_o));
      MC_API_CHECK(cudaEventRecord(ev_o, sd));
      auto jt = p->last_out.find(key);
      if (jt != p->last_out.end()) { p->live.push_back(jt->second); jt->second = ev_o; }
      else p->last_out.emplace(key, ev_o);
    }
  }
  return MC_OK;
}

// End of one host sync: `s_wait` (the caller's stream) waits for every encode and read-out
// of the call; events of this call are recycled (an event may be re-recorded once all work
// that waits on it has been enqueued, which is the case here).  s_wait = MC_PIPE_NO_WAIT
// leaves the call running: the next mc_pipe_group call overlaps it (its H2D of chunk c waits
// for this call's read-out of chunk c only) — a later mc_pipe_finish with a stream joins
// both.  (NULL is the legacy default stream, a valid s_wait.)
int mc_pipe_finish(mc_pipe* p, void* s_enc, void* s_d2h, void* s_wait) {
  if (!p) { set_error("null pipe"); return MC_EINVAL; }
  cudaStream_t se = static_cast<cudaStream_t>(s_enc), sd = static_cast<cudaStream_t>(s_d2h),
               sw = static_cast<cudaStream_t>(s_wait);
  if (!p->enc_done) MC_API_CHECK(cudaEventCreateWithFlags(&p->enc_done, cudaEventDisableTiming));
  if (!p->out_done) MC_API_CHECK(cudaEventCreateWithFlags(&p->out_done, cudaEventDisableTiming));
  MC_API_CHECK(cudaEventRecord(p->enc_done, se));
  MC_API_CHECK(cudaEventRecord(p->out_done, sd));
  if (s_wait != MC_PIPE_NO_WAIT) {
    MC_API_CHECK(cudaStreamWaitEvent(sw, p->enc_done, 0));
    MC_API_CHECK(cudaStreamWaitEvent(sw, p->out_done, 0));
    MC_API_CHECK(cudaStreamWaitEvent(se, p->out_done, 0));  // later device steps must not overwrite dev early
  }
  for (cudaEvent_t e : p->live) p->pool.push_back(e);
  p->live.clear();
  return MC_OK;
}

}  // extern "C"
