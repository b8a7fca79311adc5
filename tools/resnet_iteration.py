#!/usr/bin/env python
"""Whole synchronous-SGD iterations of ResNet-50 on synthetic ImageNet-shaped data
(the shape of PAPER.md Fig. 1 and the scaling efficiency of
PAPER.md:113-118), with the lmsgd exchange + blended update as the optimizer.

    python tools/resnet_iteration.py [--iters 30] [--warmup 5]
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/resnet_iteration.py

Per rank: minibatch 32 of 3x224x224 synthetic images, torchvision
ResNet-50 with random init, fp32 compute (cuDNN may use TF32),
BatchNorm with momentum 1.  The parameters and gradients are views
of two flat fp32 buffers (``LMSGD``, row a1), so lmsgd_step consumes the gradient in place.
Prints one JSON line on rank 0: iteration time, the exchange + update share
(the "communication time" of Fig. 1), images/s.  Forward/backward are cuDNN
(library code); the path under test is the lmsgd step.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torchvision  # noqa: E402

import paper_1711_04325_b200 as L  # noqa: E402
from paper_1711_04325_b200 import bn_sync  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--weight-decay", type=float, default=0.0, help="R12 (Goyal et al. used 1e-4)")
    ap.add_argument("--bucketed", type=int, default=0,
                    help="row f1: BucketedLMSGD with buckets of this many elements, each exchanged from a "
                         "post-accumulate-grad hook on a side stream while backward runs (0 = LMSGD, the "
                         "exchange after backward)")
    ap.add_argument("--exchange-blocks", type=int, default=0, help="bucketed: k_xstep1 grid cap (0 = whole GPU)")
    args = ap.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    torch.manual_seed(0)
    model = torchvision.models.resnet50().to(dev)
    bn_sync.last_minibatch_bn(model)
    # the torch-style front end: parameters and gradients become views of flat buffers
    if args.bucketed:
        opt = L.BucketedLMSGD(model.parameters(), cluster=L.make_cluster(1024, args.batch), loss_scale=1024.0,
                              bucket_elems=args.bucketed, exchange_blocks=args.exchange_blocks)
    else:
        opt = L.LMSGD(model.parameters(), cluster=L.make_cluster(1024, args.batch), loss_scale=1024.0,
                      weight_decay=args.weight_decay)
    n, ctx = opt.n, opt.ctx
    sync = bn_sync.BNStatsSync(model, ctx)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1711 + rank)
    x = torch.randn(args.batch, 3, 224, 224, device=dev, generator=gen)
    y = torch.randint(0, 1000, (args.batch,), device=dev, generator=gen)
    crit = torch.nn.CrossEntropyLoss()
    stream = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    fb_ms, st_ms, it_ms = [], [], []
    model.train()
    for it in range(args.warmup + args.iters):
        opt.zero_grad()
        ev[0].record(stream)
        loss = crit(model(x), y) * 1.0
        loss.backward()
        ev[1].record(stream)
        opt.step()
        ev[2].record(stream)
        torch.cuda.synchronize()
        if it >= args.warmup:
            fb_ms.append(ev[0].elapsed_time(ev[1]))
            st_ms.append(ev[1].elapsed_time(ev[2]))
            it_ms.append(ev[0].elapsed_time(ev[2]))
    code, st = opt.status()
    sync.sync()                       # BN statistics average before "validation"
    torch.cuda.synchronize()
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    res = {"fwd_bwd_ms": med(fb_ms), "exchange_update_ms": med(st_ms), "iteration_ms": med(it_ms)}
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, res)
        res = {k: max(r[k] for r in allr) for k in res}
    if rank == 0:
        out = {"what": "ResNet-50 synchronous SGD iteration, synthetic data, lmsgd exchange + update",
               "n_gpus": world, "batch_per_gpu": args.batch, "params": n, "iters": args.iters, **res,
               "optimizer": (f"BucketedLMSGD({len(opt.buckets)} buckets of ~{args.bucketed} elements, exchange "
                             f"overlapped with backward, k_xstep1 grid cap {args.exchange_blocks or 'none'})"
                             if args.bucketed else "LMSGD (lmsgd_step after backward)"),
               "note": "exchange_update_ms = backward end -> step end on the main stream: the exchange and "
                       "update time NOT hidden behind backward (with rank skew at N > 1)",
               "exchange_share": res["exchange_update_ms"] / res["iteration_ms"],
               "images_per_s": world * args.batch / (res["iteration_ms"] * 1e-3),
               "last_status": code, "loss": float(loss)}
        print(json.dumps(out), flush=True)
    opt.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
