"""One rank's sync step at N ranks, measured on ONE B200 with the other N-1 ranks simulated
(their payloads already in every gather slot and their flags already raised, as if their
pushes had landed): this rank's encode + push into the N gather buffers, then the decode of
the N gathered payloads.

  serial   mc_encode_push (end-of-kernel flags) -> mc_push_wait -> mc_decode_mean
  overlap  mc_encode_push_chunked on the sync stream || mc_decode_mean_wait on a second
           stream (chunk c decoded as soon as its flags are up, while later chunks encode)

Both on the ResNet-50 set; prints one JSON line per (codec, N, chunk).  NVLink transfer time
is not in these numbers (all slots are local HBM): the overlap step is the lower bound the
fused path reaches when the link keeps up (PUSH bytes per rank (N-1) * P at 770 GB/s:
3.2 MB x 7 = 29 us for efsignsgd at N=8, below the step)."""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2103_15195_b200 import _native, compressors as C, gradsets  # noqa: E402
from paper_2103_15195_b200.spec import CompressorSpec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--codecs", default="efsignsgd,onebit")
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--chunks", default="262144,1048576")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    gs = "resnet50_161"
    D = sum(gradsets.sizes(gs))
    x0 = torch.from_numpy(gradsets.synthetic_gradients(gs, 0, 0)).cuda()
    side = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for name in a.codecs.split(","):
        spec = CompressorSpec(name)
        L = _native.layout(spec.to_c(), D)
        stride = (L.bytes + 15) // 16 * 16
        res = torch.zeros(D, dtype=torch.float64, device="cuda") if spec.uses_error_feedback else None
        for N in map(int, a.ranks.split(",")):
            bufs = [torch.zeros(N * stride, dtype=torch.uint8, device="cuda") for _ in range(N)]
            for r in range(1, N):  # the other ranks' payloads, already gathered everywhere
                g = torch.from_numpy(gradsets.synthetic_gradients(gs, 0, r)).cuda()
                rr = torch.zeros(D, dtype=torch.float64, device="cuda") if res is not None else None
                p = C.device_encode(spec, g, rr, None, 1)
                for j in range(N):
                    bufs[j][r * stride:r * stride + L.bytes].copy_(p.buf)
            out = torch.empty(D, device="cuda")
            dsts = [b.data_ptr() for b in bufs]
            own = bufs[0][:stride]
            flags = [torch.zeros(N, dtype=torch.int32, device="cuda") for _ in range(N)]
            ep = [0]

            def serial():
                ep[0] += 1
                flags[0][1:] = ep[0]
                C.device_encode_push(spec, x0, res, None, 1, own, dsts, [f.data_ptr() for f in flags], ep[0])
                C.push_wait(flags[0], N, ep[0], err)
                C.device_decode_mean(spec, bufs[0], stride, N, D, out, err)

            def timed(fn, setup=None):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(3):
                    torch.cuda._sleep(5_000_000)
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    for _ in range(a.reps):
                        fn()
                    e.record()
                    e.synchronize()
                    best = min(best, s.elapsed_time(e) / a.reps)
                return best

            # the flag fill is a (tiny) kernel inside the timed loop in both arms
            t_serial = timed(serial)
            for target in map(int, a.chunks.split(",")):
                chunk = C.push_chunk_elems(spec, D, target)
                nch = -(-D // chunk)
                cfl = [torch.zeros(nch * N, dtype=torch.int32, device="cuda") for _ in range(N)]
                mask = torch.ones(nch, N, dtype=torch.bool, device="cuda")
                mask[:, 0] = False
                mask = mask.flatten()

                def overlap():
                    ep[0] += 1
                    cfl[0].masked_fill_(mask, ep[0])  # the other ranks' chunks have landed
                    side.wait_stream(main_s)  # before the encode: the two run at once
                    C.device_encode_push_chunked(spec, x0, res, None, 1, own, dsts, [f.data_ptr() for f in cfl], 0,
                                                 ep[0], chunk)
                    with torch.cuda.stream(side):
                        C.decode_mean_wait(spec, bufs[0], stride, N, D, out, cfl[0], chunk, ep[0], err, stream=side,
                                           timeout_s=30.0)
                    main_s.wait_stream(side)

                def push_only():
                    ep[0] += 1
                    C.device_encode_push_chunked(spec, x0, res, None, 1, own, dsts, [f.data_ptr() for f in cfl], 0,
                                                 ep[0], chunk)

                def decode_only():  # every flag already up: the waiting decode's own cost
                    cfl[0].fill_(ep[0])
                    C.decode_mean_wait(spec, bufs[0], stride, N, D, out, cfl[0], chunk, ep[0], err, timeout_s=30.0)

                t_push = timed(push_only)
                t_dec = timed(decode_only)
                t_over = timed(overlap)
                assert int(err.item()) == 0
                print(json.dumps({"codec": name, "N": N, "chunk_elems": chunk, "chunks": nch,
                                  "push_chunked_ms": round(t_push, 4), "decode_wait_ms": round(t_dec, 4),
                                  "serial_ms": round(t_serial, 4), "overlap_ms": round(t_over, 4),
                                  "serial_GBps": round(4 * D / t_serial / 1e6, 1),
                                  "overlap_GBps": round(4 * D / t_over / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
