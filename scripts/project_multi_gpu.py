"""Per-GPU sync-step time at N ranks, measured on ONE B200 for the parts this repo
owns: encode (unfused, payload only) + decode_mean over N gathered payloads (the N
payloads of N different gradient sets stacked exactly like the NCCL allgather
output).  The allgather itself is estimated from the payload size and the measured
peer bandwidth (770 GB/s per direction, B200_PROFILING.md); (N-1) * P bytes arrive
per rank.  The peer-memory path (mc_encode_push: the encode kernel stores into all N
gather slots) is measured with the N slots on this GPU and projected as
max(encode_push, allgather) + decode.  The chunk pipeline of GradSync (N > 1, per-bucket
codecs: every chunk encoded and its allgather started before the decodes) is projected
from the measured per-chunk encode (grids sized for 148 - sm_reserve SMs) and decode
times with a two-resource schedule: the SMs run E_0..E_{K-1} then D_0..D_{K-1}, the link
runs A_c = lat + (N-1) * P_c / bw after E_c (and A_{c-1}), D_c waits for A_c.  Prints one
JSON line per (codec, N)."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_15195_b200 import compressors as C, gradsets  # noqa: E402
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402


def timed(fn, reps=20, trials=3):
    """Device time per call: a ~5 ms spin kernel keeps the GPU busy while the host enqueues
    all reps, so host launch overhead never shows up as GPU idle time between the events.
    Minimum over `trials` (a host stall longer than the spin would leave the GPU idle)."""
    for _ in range(3):
        fn()
    best = float("inf")
    for _ in range(trials):
        torch.cuda.synchronize()
        torch.cuda._sleep(10_000_000)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / reps)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gradset", default="resnet50_161")
    ap.add_argument("--codecs", default="efsignsgd,onebit,dgc_lite,qsgd,terngrad,int8,fp16")
    ap.add_argument("--nccl-lat-us", type=float, default=10.0,
                    help="per-call allgather latency added to bytes / 770 GB/s (assumed, not measured here)")
    ap.add_argument("--sm-reserve", type=int, default=16)
    a = ap.parse_args()
    lat = a.nccl_lat_us * 1e-3
    from paper_2103_15195_b200 import _native
    from paper_2103_15195_b200.sync import GradSync
    D = sum(gradsets.sizes(a.gradset))
    grads = [torch.from_numpy(gradsets.synthetic_gradients(a.gradset, 0, r)).cuda() for r in range(8)]
    for name in a.codecs.split(","):
        spec = CompressorSpec(name, sparsity=0.999 if name in ("topk", "dgc_lite") else 0.99)
        res = torch.zeros(D, dtype=torch.float64, device="cuda") if spec.uses_error_feedback else None
        pays = [C.device_encode(spec, g, None if res is None else res.clone(), None, 1) for g in grads]
        stride = pays[0].buf.numel()
        gathered = torch.cat([p.buf for p in pays])
        out = torch.empty(D, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        x = grads[0].clone()
        t_enc = timed(lambda: C.device_encode(spec, x, res, None, 1, out=pays[0].buf))
        P = C.payload_bytes(spec, D)
        for N in (1, 2, 4, 8):
            t_dec = timed(lambda: C.device_decode_mean(spec, gathered, stride, N, D, out, err))
            t_ag = (lat if N > 1 else 0.0) + (N - 1) * P / 770e9 * 1e3
            step = t_enc + t_ag + t_dec
            # fused encode + push (mc_encode_push) into N gather buffers of this GPU: the kernel
            # cost of storing into every slot; over NVLink the (N-1)*P bytes need t_ag, which
            # the push overlaps with the encode, so the p2p step is max(encode_push, t_ag) + decode
            pstride = (stride + 15) // 16 * 16
            bufs = [torch.zeros(N * pstride, dtype=torch.uint8, device="cuda") for _ in range(N)]
            flg = [torch.zeros(N, dtype=torch.int32, device="cuda") for _ in range(N)]
            ep = [0]

            def push():
                ep[0] += 1
                C.device_encode_push(spec, x, res, None, 1, bufs[0][:pstride], [b.data_ptr() for b in bufs],
                                     [f.data_ptr() for f in flg], ep[0])

            t_push = timed(push)
            step_p2p = max(t_push, t_ag) + t_dec
            chunk = {}
            if name in GradSync.CHUNKABLE and N > 1:
                K = max(1, min(4, D // GradSync.CHUNK_MIN))
                B = spec.bucket_size
                al = B * 32 // __import__("math").gcd(B, 32)
                tgt = -(-(-(-D // K)) // al) * al
                bounds = [(c, min(D, c + tgt)) for c in range(0, D, tgt)]
                lib = _native.lib()
                prev = lib.mc_set_sm_reserve(a.sm_reserve)
                try:
                    e_t, d_t, a_t = [], [], []
                    for c0, c1 in bounds:
                        nc = c1 - c0
                        xc = x[c0:c1]
                        rc = None if res is None else res[c0:c1]
                        pc = C.device_encode(spec, xc, rc, None, 1)
                        e_t.append(timed(lambda: C.device_encode(spec, xc, rc, None, 1, out=pc.buf)))
                        gc = torch.cat([pc.buf] * N)
                        oc = out[c0:c1]
                        d_t.append(timed(lambda: C.device_decode_mean(spec, gc, pc.buf.numel(), N, nc, oc, err)))
                        a_t.append(lat + (N - 1) * C.payload_bytes(spec, nc) / 770e9 * 1e3)
                finally:
                    lib.mc_set_sm_reserve(prev)
                t_sm, t_link, e_end = 0.0, 0.0, []
                for c in range(len(bounds)):
                    t_sm += e_t[c]
                    e_end.append(t_sm)
                a_end = []
                for c in range(len(bounds)):
                    t_link = max(t_link, e_end[c]) + a_t[c]
                    a_end.append(t_link)
                for c in range(len(bounds)):
                    t_sm = max(t_sm, a_end[c]) + d_t[c]
                chunk = {"chunks": len(bounds), "chunk_encode_ms": round(sum(e_t), 4),
                         "chunk_decode_ms": round(sum(d_t), 4), "chunk_allgather_ms": round(sum(a_t), 4),
                         "chunk_step_ms": round(t_sm, 4), "chunk_per_gpu_GBps": round(4 * D / t_sm / 1e6, 1),
                         "nccl_lat_us_assumed": a.nccl_lat_us}
            print(json.dumps({"codec": name, "N": N, "encode_ms": round(t_enc, 4), "decode_mean_ms": round(t_dec, 4),
                              "allgather_est_ms": round(t_ag, 4), "step_ms": round(step, 4),
                              "per_gpu_GBps": round(4 * D / step / 1e6, 1), "encode_push_ms": round(t_push, 4),
                              "p2p_step_ms": round(step_p2p, 4),
                              "p2p_per_gpu_GBps": round(4 * D / step_p2p / 1e6, 1), **chunk}), flush=True)


if __name__ == "__main__":
    main()
