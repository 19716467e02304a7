"""Batched TT rounding micro-benchmark: `count` CTAs each round the same
FFT-product-shaped TT (ttgbf_tt_round, one launch), the rounding load of the
bench's FFT-convolution stage without its cross noise -- a deterministic A/B
for rounding changes.

  python tools/round_batch_bench.py [--ranks 1,100,160,180,280,100,1] [--n 65] [--count 296]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--ranks", default="1,100,160,180,280,100,1")
    p.add_argument("--n", type=int, default=65)
    p.add_argument("--count", type=int, default=296)
    p.add_argument("--reps", type=int, default=3)
    p.add_argument("--cap", type=int, default=20)
    p.add_argument("--ws-mb", type=int, default=200)
    a = p.parse_args()
    import torch
    from paper_2501_07942_b200 import _abi
    from paper_2501_07942_b200.backend import CudaBackend
    from tools.round_bench import qr_flops
    be = CudaBackend()
    lib = be.lib
    ranks = [int(x) for x in a.ranks.split(",")]
    d = len(ranks) - 1
    rs = np.random.RandomState(0)
    cores = []
    for k in range(d):
        c = rs.randn(ranks[k], a.n, ranks[k + 1])
        c *= (0.9 ** np.arange(ranks[k + 1]))[None, None, :]
        cores.append(c)
    h = np.zeros(a.count, dtype=_abi.TT)
    off = 0
    for k, c in enumerate(cores):
        h["n"][:, k] = a.n
        h["r"][:, k] = c.shape[0]
        h["off"][:, k] = off
        off += c.size
    h["r"][:, d] = 1
    h["d"] = d
    size = off
    flat = np.concatenate([c.reshape(-1) for c in cores])
    src = torch.from_numpy(np.tile(flat, a.count)).to(be.device)
    hin = be.upload(h)
    hout = be.empty(a.count * _abi.TT.itemsize)
    out_cap = sum(a.n * min(r, a.cap) ** 2 for r in ranks) + 16
    out = torch.empty(a.count * out_cap, dtype=torch.float64, device=be.device)
    ws_bytes = a.ws_mb << 20
    ws = be.empty(a.count * ws_bytes)
    st = be.empty(4 * a.count)
    work = torch.empty_like(src)
    ts = []
    for rep in range(a.reps + 1):
        work.copy_(src)    # rounding destroys nothing in the input, but keep the same bytes
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.ttgbf_tt_round(hin.ptr, work.data_ptr(), size, a.count, 1e-8, a.cap, hout.ptr, out.data_ptr(),
                                out_cap, ws.ptr, ws_bytes, st.ptr, be.stream_ptr)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0
        if rep:
            ts.append(e0.elapsed_time(e1) / 1e3)
    status = be.download(st, np.int32, a.count)
    ho = be.download(hout, _abi.TT, a.count)
    fl = qr_flops(ranks, a.n) * a.count
    t = min(ts)
    print(json.dumps({"ranks": ranks, "n": a.n, "count": a.count, "seconds": t, "qr_gflop": fl / 1e9,
                      "qr_tflops": fl / t / 1e12, "status_ok": int((status == 0).sum()),
                      "out_ranks": [int(v) for v in ho[0]["r"][: d + 1]]}))


if __name__ == "__main__":
    main()
