"""BASELINE configs[4] batch-sharded: the sparsity sweep on ResNet-50 layer shapes at a
global batch of 1024, split over N ranks (one per GPU) with sharding.ShardedRun
(strong scaling: the same 1024 images whatever N), each point with its committed tile
(profiles/r02_tuned_sweep.json).  Per point: device time of each rank's launch (CUDA
events, max over ranks) and global images/s; after timing, the final gather
(all_gather of the outputs) is run once and rank 0 checks sample rows from every rank's
shard against the single-device launch of the same rows.

    python tools/sweep_sharded.py [--gpus N] [--points r50-1x1-64x256-32@0.9,...]

Without a torchrun environment, --gpus N re-launches under torch.distributed.run.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

SHAPES = {"r50-3x3-64x32": (64, 64, 3, 32), "r50-3x3-256x8": (256, 256, 3, 8),
          "r50-1x1-64x256-32": (64, 256, 1, 32), "r50-1x1-256x64-32": (256, 64, 1, 32)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--points", default=None)
    ap.add_argument("--global-batch", type=int, default=1024)
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and (args.gpus or 1) > 1:
        import bench
        bench.launch_ranks(args, __file__)  # re-exec under torchrun (same contract as bench.py)
    import torch
    import torch.distributed as dist
    import paper_2112_15445_b200 as U
    from paper_2112_15445_b200 import _lib
    from paper_2112_15445_b200.engine import ExecConfig, launch, padded_input, plan_for
    from paper_2112_15445_b200.pruning import synthesize_masked_weights
    rank, local, world = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("LOCAL_RANK", 0), ("WORLD_SIZE", 1)))
    if args.gpus is not None and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but {world} rank(s) launched")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    job = U.ShardedRun.from_env(args.global_batch, align=64)
    tiles = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_sweep.json")))
    keys = args.points.split(",") if args.points else list(tiles)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    for key in keys:
        name, s = key.split("@")
        c, d, k, hw = SHAPES[name]
        g = U.ConvGeometry(c, d, k, k, hw, hw, padding=(k // 2, k // 2))
        w = synthesize_masked_weights(g, float(s), np.random.default_rng([0, int(float(s) * 1000)]))
        f = U.build_csr(w, g)
        rng = np.random.default_rng([5, c, d, hw])
        x_all = rng.standard_normal((args.global_batch, c, hw, hw)).astype(np.float32)
        xl = torch.from_numpy(np.ascontiguousarray(job.local(x_all))).cuda()
        n = job.local_batch
        plan, blob = plan_for(f, n, _lib.USC_F32, ExecConfig(**tiles[key]), f.weights)
        xp = padded_input(xl, plan)
        lay = _lib.act_layout(d, g.out_h, g.out_w, 1, 1, 4, plan.in_.interleave)
        y = torch.zeros(lay.elems(n), dtype=torch.float32, device="cuda")
        epi = _lib.Epilogue()
        epi.scale, epi.out_padded, epi.out = 1.0, 1, lay
        for _ in range(3):
            launch(plan, blob, xp, y, epi)
        ts = []
        for _ in range(9):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            a.record()
            launch(plan, blob, xp, y, epi)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        # the final gather, once: unpack this rank's rows and all_gather them
        out = torch.empty((n, d, g.out_h, g.out_w), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().usc_unpad_output(_lib.ref(lay), _lib.USC_F32, n, _lib.t_ptr(y), _lib.t_ptr(out),
                                               _lib.stream_ptr()))
        full = job.gather(out)
        ok = None
        if rank == 0:
            rows = np.unique(np.r_[0, 1, args.global_batch // 2, args.global_batch - 1])
            xr = torch.from_numpy(np.ascontiguousarray(x_all[rows])).cuda()
            ref = U.sparse_conv_forward(U.DenseTensor4(xr), f, ExecConfig(**tiles[key])).device()
            ok = bool(torch.equal(full[rows], ref))
            print(json.dumps({"point": key, "n_gpus": world, "global_batch": args.global_batch,
                              "per_rank_batch": n, "us_max_over_ranks": round(ms * 1e3, 1),
                              "images_per_s": round(args.global_batch / (ms / 1e3), 1),
                              "scaling": "strong", "gathered_rows_bitwise": ok}), flush=True)
        f._packs.clear()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
