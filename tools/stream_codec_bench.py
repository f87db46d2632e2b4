"""Throughput of the streaming-exponent BFP codec (N3) against the fixed-block
codec on one GPU: n = 2^27 doubles, CUDA events on the current stream, L2
flushed between repetitions.  Algorithmic bytes: encode 8n read + n w / 8
written; decode the reverse."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2511_19036_b200 as P
from fmg_inputs import codec_vectors


def timed(fn, reps=10):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(reps + 2):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts[2:])[len(ts[2:]) // 2]


def main():
    n = 1 << 27
    out = {"n": n}
    for kind in ("smooth", "staircase"):
        x = torch.from_numpy(codec_vectors(n, seed=5, kind=kind)).cuda()
        for w in (4, 8, 16):
            mant, xe, xs, nb = P.bfp_stream_encode(x, w)
            t_se = timed(lambda: P.bfp_stream_encode(x, w))
            t_sd = timed(lambda: P.bfp_stream_decode(mant, xe, xs, nb, n, w))
            assert P.bfp_status() == 0
            gb = (8 * n + n * w / 8) / 1e9
            r = {"stream_encode_ms": t_se, "stream_decode_ms": t_sd,
                 "stream_encode_GBs": gb / t_se * 1e3, "stream_decode_GBs": gb / t_sd * 1e3,
                 "nblocks": int(nb.item())}
            if kind == "smooth":  # the int8-exponent block codec rejects the staircase range
                m2, e2 = P.bfp_encode(x, w)
                t_be = timed(lambda: P.bfp_encode(x, w))
                t_bd = timed(lambda: P.bfp_decode(m2, e2, n, w))
                assert P.bfp_status() == 0
                r.update({"block_encode_ms": t_be, "block_decode_ms": t_bd,
                          "block_encode_GBs": (gb + n / 32 / 1e9) / t_be * 1e3,
                          "block_decode_GBs": (gb + n / 32 / 1e9) / t_bd * 1e3})
            out[f"{kind}_w{w}"] = r
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
