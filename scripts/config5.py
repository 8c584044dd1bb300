#!/usr/bin/env python3
"""Config 5: 3-D 27-point stencil g^3 (default 512^3: 134M rows, 3.6e9 nnz),
row-partitioned iterated DIA SpMV with halo exchange over NVLink (NCCL
point-to-point through torch.distributed), 1/2/4/8 GPUs.

Each rank generates only its row slice on its own device
(so_gen_stencil27_dia), keeps x on its window, and runs
paper_2303_05098_b200.dist.iterate: boundary rows, halo isend/irecv, interior
rows overlapping the exchange.  Timed with CUDA events on the launching
stream, max over ranks; prints one JSON line on rank 0.

    python scripts/config5.py --g 512 --iters 20
    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 scripts/config5.py
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_05098_b200 as P  # noqa: E402
from paper_2303_05098_b200 import dist as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--g", type=int, default=512)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="p2p: boundary rows pushed into the neighbours' windows by the multiply "
                         "(so_spmv_rows_push over CUDA IPC); nccl: isend/irecv after the multiply")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    P.set_device(local)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    g = a.g
    n = g ** 3
    h = g * g + g + 1
    s = D.partition(n, h, rank, world)
    m = P.DeviceMatrix.stencil27(g, s.r0, s.r1, s.w0, s.w1, seed=5)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    idx = torch.arange(s.w0, s.w1, dtype=torch.int64, device="cuda")
    xa = 1.0 + (idx % 7).to(torch.float64) / 8.0
    xb = torch.zeros_like(xa)
    del idx

    def spmv_rows(xw, yw, lo, hi):
        m.spmv_device_rows(xw.data_ptr(), yw.data_ptr() + 8 * s.own_lo, lo, hi, stream.cuda_stream)

    def exchange(buf, plan):
        if world == 1:
            return None
        reqs = []
        for peer, (sa, sb), (ra, rb) in plan:
            reqs.append(torch.distributed.isend(buf[sa:sb], peer))
            reqs.append(torch.distributed.irecv(buf[ra:rb], peer))

        def wait():
            for r in reqs:
                r.wait()
        return wait

    it = D.make_iterator(s, m, torch.distributed if world > 1 else None, a.exchange, stream) if world > 1 else None
    if it is not None:
        it.load_x(lambda lo, hi: 1.0 + (torch.arange(lo, hi, dtype=torch.int64, device="cuda") % 7).double() / 8.0)
        del xa, xb
        torch.cuda.synchronize()
        torch.distributed.barrier()
        it.run(a.warmup)
    else:
        out = D.iterate(s, xa, xb, a.warmup, spmv_rows, exchange)
        other = xb if out is xa else xa
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if it is not None:
        it.run(a.iters)
    else:
        out = D.iterate(s, out, other, a.iters, spmv_rows, exchange)
    e1.record(stream)
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) * 1e-3 / a.iters
    t = torch.tensor([sec, float(m.spmv_bytes)], dtype=torch.float64, device="cuda")
    if world > 1:
        tmax = t.clone()
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tsum = t.clone()
        torch.distributed.all_reduce(tsum, op=torch.distributed.ReduceOp.SUM)
        sec, nbytes = float(tmax[0]), float(tsum[1])
    else:
        sec, nbytes = float(t[0]), float(t[1])
    # checksum of the final iterate's owned rows (identical for every P)
    csum = it.checksum() if it is not None else D.owned_checksum(out[s.own_lo:s.own_hi], s)
    if rank == 0:
        peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
        print(json.dumps({"metric": "spmv_gbs_iterated", "config": f"27-pt stencil {g}^3 DIA, row-partitioned",
                          "n_gpus": world, "nrows": n, "iters": a.iters, "ms_per_iter": round(sec * 1e3, 4),
                          "value": round(nbytes / sec / 1e9, 1), "unit": "GB/s",
                          "frac_per_gpu": round(nbytes / sec / 1e9 / world / peak, 4),
                          "halo_rows_per_side": h, "exchange": a.exchange if world > 1 else "none",
                          "checksum": csum}), flush=True)
    if world > 1:
        torch.distributed.barrier()
        if it is not None:
            it.close()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
