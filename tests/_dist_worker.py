"""Worker for tests/test_gpu_parity.py::test_sharded_ranks_share_gpu: one rank of
the sharded count (paper_1608_05138_b200.dist.count_sharded) with every rank on
cuda:0 and gloo collectives, so the multi-rank path runs on a one-GPU box.
Writes its micro-record shard and X to <out>/rank<r>.npy / .json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def make_pairs(gl, spec):
    """rmat:<scale> (seed 3) or ba:<n>:<k>:<seed>"""
    kind, *a = spec.split(":")
    if kind == "rmat":
        return gl.generate_rmat(int(a[0]), 16, seed=3)
    return gl.generate_ba(int(a[0]), int(a[1]), seed=int(a[2]))


def main(out_dir, spec):
    import torch
    import torch.distributed as dist
    import paper_1608_05138_b200 as gl
    from paper_1608_05138_b200.dist import count_sharded
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    g = gl.Graph.build(make_pairs(gl, spec), 0)
    X, (b, e) = count_sharded(g, rank, world)
    rec = g.micro_records(b, e - b) if e > b else np.zeros(0, gl.MICRO_DTYPE)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), rec)
    json.dump({"X": [str(x) for x in X], "b": b, "e": e}, open(os.path.join(out_dir, f"rank{rank}.json"), "w"))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
