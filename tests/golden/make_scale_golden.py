"""Full-size parity fixtures from the REFERENCE's own code (oracle/_ref).

TEST INFRASTRUCTURE.  Graphs come from the oracle's ports of the product's
deterministic generators (oracle.c or_generate_rmat / or_generate_ba, pinned
equal to the product's by tests/test_oracle.py), so no product code is loaded.

  full   <spec>   every edge through the reference pipeline (ref_count:
                  process_edge_hash + accumulate_unrestricted + merge +
                  global_from_unrestricted, kernels.cpp:143-156,
                  counts.cpp:6-111): X_1..X_17, sha256 of the whole MicroRecord
                  table (m x 10 little-endian u64, counts.hpp:82-89 field
                  order, edge-id order) and of the oriented-edge label table
                  -> tests/golden/full_<name>.json
  sample <spec>   stratified edge sample through process_edge_hash: the
                  --heavy edges of largest d_u + d_v plus --uniform uniformly
                  drawn edge ids -> tests/golden/sample_<name>.npz (ids and
                  {v label, u label, t, s_u, s_v, x7, x10} rows) + .json header

spec: rmat:<scale>[:<seed>]  (edge factor 16, a,b,c = .57,.19,.19; seed 1)
      ba:<n>:<attach>[:<seed>]
Run where the reference sources compiled (this container) or on a box with
the prebuilt oracle/_ref; wall time is recorded in the output.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402


def make_pairs(spec: str):
    kind, *a = spec.split(":")
    if kind == "rmat":
        scale, seed = int(a[0]), int(a[1]) if len(a) > 1 else 1
        return O.generate_rmat(scale, 16, seed=seed), f"rmat{scale}_s{seed}", {
            "generator": "rmat", "scale": scale, "edge_factor": 16, "a": 0.57, "b": 0.19, "c": 0.19, "seed": seed}
    if kind == "ba":
        n, k, seed = int(a[0]), int(a[1]), int(a[2]) if len(a) > 2 else 1
        return O.generate_ba(n, k, seed=seed), f"ba{n}_{k}_s{seed}", {
            "generator": "ba", "n": n, "attach": k, "seed": seed}
    raise SystemExit(f"bad spec {spec}")


def label_digest(ref) -> str:
    v, u, vl, ul = ref.orient()
    return hashlib.sha256(np.stack([vl, ul], axis=1).astype("<u8").tobytes()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["full", "sample"])
    ap.add_argument("spec")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--heavy", type=int, default=2000)
    ap.add_argument("--uniform", type=int, default=100000)
    ap.add_argument("--out", default=HERE)
    args = ap.parse_args()
    if not O.ref_available():
        raise SystemExit("oracle/_ref missing: make -C oracle ref")
    t0 = time.time()
    pairs, name, gen = make_pairs(args.spec)
    t1 = time.time()
    ref = O.RefLib(pairs)
    del pairs
    t2 = time.time()
    n, m = ref.n, ref.m
    head = {"spec": args.spec, "graph": gen, "n": n, "m": m, "source": "oracle/_ref (reference sources compiled in place)",
            "edge_labels_sha256": label_digest(ref), "threads": args.threads,
            "seconds": {"generate": round(t1 - t0, 1), "reference_build": round(t2 - t1, 1)}}
    print(f"[golden] {name}: n={n} m={m} build {t2 - t1:.1f}s", flush=True)
    if args.mode == "full":
        X, rec = ref.count(threads=args.threads, micro=True)
        head["seconds"]["reference_count"] = round(time.time() - t2, 1)
        head["X"] = [str(x) for x in X]
        head["micro_sha256"] = hashlib.sha256(np.ascontiguousarray(rec).view("<u8").tobytes()).hexdigest()
        path = os.path.join(args.out, f"full_{name}.json")
    else:
        v, u, _, _ = ref.orient()
        deg = ref.degrees().astype(np.uint64)
        w = deg[v] + deg[u]
        heavy = np.argsort(-w.astype(np.int64), kind="stable")[: min(args.heavy, m)].astype(np.uint64)
        rng = np.random.default_rng(12345)
        uni = np.sort(rng.choice(m, size=min(args.uniform, m), replace=False)).astype(np.uint64)
        ids = np.unique(np.concatenate([heavy, uni]))
        rows = ref.edges(ids, threads=args.threads)
        head["seconds"]["reference_edges"] = round(time.time() - t2, 1)
        head["n_heavy"], head["n_uniform"], head["n_ids"] = int(len(heavy)), int(len(uni)), int(len(ids))
        head["sample"] = (f"{len(heavy)} edges of largest d_u+d_v plus {len(uni)} uniform edge ids "
                          "(numpy default_rng(12345)), through process_edge_hash")
        path = os.path.join(args.out, f"sample_{name}.npz")
        np.savez_compressed(path, ids=ids, rows=rows)
        path = os.path.join(args.out, f"sample_{name}.json")
    with open(path, "w") as f:
        json.dump(head, f, indent=1)
    print(f"[golden] wrote {path} ({time.time() - t0:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
