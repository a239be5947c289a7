"""One rank of tests/test_gpu_nccl.py (launched by torch.distributed.run, NCCL backend,
one GPU per rank): generate only this rank's groups (per-group seeds), run the kernel
on them slab by slab with the output all-gathered per slab over NCCL on a side stream
(distributed.SlabGather), and on rank 0 compare the gathered batch with one launch over
the whole batch on that GPU. Prints one JSON line on rank 0."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2412_03594_b200 import distributed as D  # noqa: E402
from paper_2412_03594_b200 import packed as P  # noqa: E402
from paper_2412_03594_b200 import workloads as W  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    spec = W.config(sys.argv[1] if len(sys.argv) > 1 else "c4")
    off = W.offsets(spec)
    shards = D.shard(off["cu_req"], off["cu_q"], off["cu_prefix"], off["cu_distinct"], spec.Hq,
                     spec.Hkv, spec.d, spec.dv, spec.torch_dtype, world)
    me = shards[rank]
    sub = spec.subset(me.groups.tolist())
    b = W.make_batch(sub, dev)  # this rank's groups only
    sg = D.SlabGather(shards, rank, 3, (spec.Hq, spec.dv), spec.torch_dtype, dev)
    ops = {}

    def compute(i, out_rows):
        g0, g1 = sg.slab_groups(i)
        r0, r1 = int(b["cu_req"][g0]), int(b["cu_req"][g1])
        t0, t1 = int(b["cu_q"][r0]), int(b["cu_q"][r1])
        p0, p1 = int(b["cu_prefix"][g0]), int(b["cu_prefix"][g1])
        d0, d1 = int(b["cu_distinct"][r0]), int(b["cu_distinct"][r1])
        if i not in ops:
            ops[i] = P.PrefixSharedAttention(
                b["cu_req"][g0:g1 + 1] - r0, b["cu_q"][r0:r1 + 1] - t0,
                b["cu_prefix"][g0:g1 + 1] - p0, b["cu_distinct"][r0:r1 + 1] - d0,
                spec.Hq, spec.Hkv, spec.d, spec.dv, spec.torch_dtype, dev)
        ops[i](b["q"][t0:t1], b["k_prefix"][p0:p1], b["v_prefix"][p0:p1], b["k_distinct"][d0:d1],
               b["v_distinct"][d0:d1], out=out_rows)

    sg.run(compute)
    out = sg.result()
    torch.cuda.synchronize()
    errs = [op.device_error() for op in ops.values()]
    if rank == 0:
        fb = W.make_batch(spec, dev)
        full = P.prefix_shared_attention_packed(fb["q"], fb["k_prefix"], fb["v_prefix"],
                                                fb["k_distinct"], fb["v_distinct"], fb["cu_req"],
                                                fb["cu_q"], fb["cu_prefix"], fb["cu_distinct"],
                                                spec.Hkv)
        torch.cuda.synchronize()
        print(json.dumps({"world": world, "rows": int(out.shape[0]), "nan": bool(torch.isnan(out).any()),
                          "max_abs_diff": float((out.float() - full.float()).abs().max()),
                          "device_errors": errs}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
