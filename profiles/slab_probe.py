"""Per-rank work of the theta-slab sharded top-level search, measured on ONE
GPU: the device-resident slab search (`search_top_slab_async`) of slab g of G
for G in {1, 2, 4, 8}, steps enqueued back to back with an L2 flush between
them, CUDA events on the library's stream.  This is the compute a rank does at
N = G (the NCCL all-gather of k x 40 B rows and the device merge are not
included: they need G GPUs), so `projected_scaling = t(G=1) / max_g t(g of G)`
is an upper bound of the bench's strong scaling, labelled as a projection.

    python profiles/slab_probe.py [--config cfg2] [--steps 50]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2112_05576_b200 as ea  # noqa: E402
from paper_2112_05576_b200 import parallel  # noqa: E402


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--sizes", default="", help="theta-slab sizes [0, s) instead of worlds")
    ap.add_argument("--no-flush", action="store_true", help="no L2 flush between steps")
    ap.add_argument("--preblock", type=float, default=0.0,
                    help="ms of GPU sleep before the timed loop (host gets ahead)")
    args = ap.parse_args()

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = ea.Context(0)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_timing(True)
    img, tmpl, cfg, _ = bench.make_inputs(args.config)
    det = ea.Detector(tmpl, cfg, ctx)
    det.levels.set_image(img)
    tg = bench.top_grid(cfg)
    nx, ny, nt = ea.grid_counts(tg)
    n_top = len(det.levels.model(cfg.num_levels - 1).points)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rows = torch.empty((cfg.topk, 5), dtype=torch.float64, device=dev)

    out = {"config": args.config, "grid": f"{nx}x{ny}x{nt}", "n_top": n_top, "slabs": {}}
    plans = ([(s, [(0, int(s))]) for s in args.sizes.split(",")] if args.sizes else
             [(G, [parallel.theta_slab(nt, g, int(G)) for g in range(int(G))])
              for G in args.worlds.split(",")])
    for G, slabs in plans:
        G = int(G)
        worst = None
        allrec = []
        for it0, it1 in slabs:
            for _ in range(args.warmup):
                ea.search_top_slab_async(det.levels, cfg, it0, it1, rows.data_ptr())
            torch.cuda.synchronize()
            ea.async_status(ctx)
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(args.steps)]
            if args.preblock:  # host runs ahead: device times exclude enqueue gaps
                torch.cuda._sleep(int(args.preblock * 1.9e6))
            h0 = time.perf_counter()
            for i in range(args.steps):
                if not args.no_flush:
                    flush.zero_()
                ev[i][0].record(stream)
                ea.search_top_slab_async(det.levels, cfg, it0, it1, rows.data_ptr())
                ev[i][1].record(stream)
            host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
            torch.cuda.synchronize()
            _, times = ea.async_status(ctx)
            step = statistics.median(a.elapsed_time(b) for a, b in ev)
            scr = statistics.median(times) if times else None
            ea.search_top_slab(det.levels, cfg, it0, it1)  # synchronous: fills the stats
            st = ctx.stats()
            rec = {"slab": [it0, it1], "step_ms": step, "screen_ms": scr, "host_enqueue_ms": host_ms,
                   "other_ms": step - scr if scr is not None else None,
                   "candidates": st["candidates"], "threshold": st["threshold"]}
            allrec.append((round(step, 4), round(scr, 4) if scr else None))
            if worst is None or step > worst["step_ms"]:
                worst = rec
        worst["all_step_screen_ms"] = allrec
        out["slabs"][G] = worst
    t1 = out["slabs"][1]["step_ms"] if 1 in out["slabs"] and not args.sizes else None
    for G, rec in out["slabs"].items():
        rec["projected_scaling"] = t1 / rec["step_ms"] if t1 else None
    print(json.dumps(out))


if __name__ == "__main__":
    main()
