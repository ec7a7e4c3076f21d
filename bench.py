#!/usr/bin/env python
"""Benchmark: edges/s for all k<=4 graphlets (macro + micro) on B200.

Workload (BASELINE.json configs[1]): RMAT scale 20, edge factor 16
(Graph500 a,b,c = .57,.19,.19, seed 1) -> 16.8M generated pairs, 15.7M unique
undirected edges, 1M vertex labels.  Synthetic, generated in HBM by the
library's own counter-based generator (identical to the host generator).

One step = one full count of the device-resident preprocessed graph: per-edge
triangles, clique and cycle kernels, per-edge epilogue + 128-bit macro
reduction (every edge's micro record t/x7/x10 is produced in HBM) and the
host-side X_1..X_17 algebra.  value = m * steps / sum of per-step device time
(CUDA events on the launching stream); L2 is flushed before every step with a
256 MiB write (outside the events).  N>1: one process per GPU, graph
replicated, cost-balanced work shares, one reduce-scatter of the per-edge
partial rows + one all-reduce of the macro sums (NCCL), time = max over ranks.

e2e: the same metric through the public C-ABI from pinned HOST pairs:
gl_graph_build (H2D + on-device CSR build) + count + D2H of every edge's
(t, x7, x10) and the macro vector, wall-clocked per step.

--impl reference: the reference's own CPU path (oracle/_ref, compiled from
/root/reference/proj/src: process_edge_hash + accumulate_unrestricted with all
host threads) on a uniform random sample of the same graph's edges.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges/sec for all k=4 graphlets (macro+micro), 1/2/4/8 B200, % HBM roofline"
UNIT = "edges/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--graph", choices=["rmat", "ba"], default="rmat",
                    help="rmat: configs[1]/[3]/[4] (RMAT/Kronecker scale S); ba: configs[2] (Barabasi-Albert)")
    ap.add_argument("--scale", type=int, default=20)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--ba-n", type=int, default=4_000_000)
    ap.add_argument("--ba-attach", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-text-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--e2e-warmup", type=int, default=5)  # the pool and pinned pages settle after ~4 e2e steps
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload(args):
    if args.graph == "ba":
        return {"workload": f"Barabasi-Albert n={args.ba_n} attach={args.ba_attach} (seed {args.seed}), "
                            "k=4 macro+micro", "ba_n": args.ba_n, "ba_attach": args.ba_attach}
    return {"workload": f"RMAT scale-{args.scale} (2^{args.scale} vertex labels, edge factor {args.edge_factor}, "
                        f"a,b,c=.57,.19,.19, seed {args.seed}), k=4 macro+micro",
            "scale": args.scale, "edge_factor": args.edge_factor}


def workload_key(args):
    """Key of this workload in profiles/traffic.json (ncu DRAM bytes per workload)."""
    if args.graph == "ba":
        return f"ba{args.ba_n}_{args.ba_attach}_s{args.seed}"
    return f"rmat{args.scale}_ef{args.edge_factor}_s{args.seed}"


def host_pairs(args):
    import paper_1608_05138_b200 as gl
    if args.graph == "ba":
        return gl.generate_ba(args.ba_n, args.ba_attach, seed=args.seed)
    return gl.generate_rmat(args.scale, args.edge_factor, seed=args.seed)


def oracle_pairs(args):
    """The same pairs from the oracle's generator ports (oracle.c, pinned equal
    to the product's generators by tests/test_oracle.py): the reference arm
    never loads the product library."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # CPU checker / baseline only
    if args.graph == "ba":
        return O.generate_ba(args.ba_n, args.ba_attach, seed=args.seed)
    return O.generate_rmat(args.scale, args.edge_factor, seed=args.seed)


# --------------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self):
        if self.p is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- reference

def ref_checker():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O  # CPU checker / baseline only
    if O.ref_available():
        return O.RefLib, "reference", "oracle/_ref (reference sources compiled in place)"
    return O.Oracle, "port", "oracle/liboracle.so (C restatement)"


def cpu_sample_run(pairs, seconds, seed=0, threads=None, steps=1):
    """Time the reference CPU path on uniform random edge samples; returns
    (edges/s per step list, cores, kind, sample description)."""
    Cls, kind, what = ref_checker()
    threads = threads or os.cpu_count() or 1
    t0 = time.time()
    ref = Cls(pairs)
    build_s = time.time() - t0
    m = ref.m
    rng = np.random.default_rng(seed)
    calib = np.sort(rng.choice(m, size=min(m, 32 * threads), replace=False)).astype(np.uint64)
    secs, _ = ref.time_sample(calib, threads)
    per_edge = max(secs / max(1, len(calib)), 1e-9)
    k = int(min(m, max(len(calib), seconds / per_edge)))
    rates = []
    for s in range(steps):
        ids = np.sort(rng.choice(m, size=k, replace=False)).astype(np.uint64)
        secs, _ = ref.time_sample(ids, threads)
        rates.append(k / secs)
    desc = (f"{k} uniformly sampled edges (of m={m}) per step through {what}: process_edge_hash + "
            f"accumulate_unrestricted, {threads} threads; graph build {build_s:.1f}s untimed")
    return rates, threads, kind, desc


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    pairs = oracle_pairs(args)
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    rates, cores, kind, desc = cpu_sample_run(pairs, per_step, steps=args.steps + args.warmup)
    rates = rates[args.warmup:] or rates
    value = statistics.mean(rates)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic", "impl": "reference",
            "config": workload(args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------- ours

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1608_05138_b200 as gl
    from paper_1608_05138_b200.dist import shard_range, sharded_step

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # GL_BENCH_SHARE_GPU=1 (test hook): every rank on cuda:0 with the gloo backend,
    # to exercise the sharded path on a one-GPU box; production runs use NCCL, one GPU per rank
    share = os.environ.get("GL_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- input generated in HBM (RMAT) or on the host (BA), CSR built on device (untimed setup)
    hp = None
    if args.graph == "ba":
        hp = host_pairs(args)
        count = len(hp)
        d_pairs = torch.from_numpy(hp.view(np.int64).reshape(-1)).to(dev)
    else:
        count = args.edge_factor << args.scale
        d_pairs = torch.empty(2 * count, dtype=torch.int64, device=dev)
        gl.generate_rmat_device(args.scale, args.edge_factor, d_pairs.data_ptr(), local, seed=args.seed)
    torch.cuda.synchronize()
    tb = time.perf_counter()
    g = gl.Graph.build_device(d_pairs.data_ptr(), count, local)
    build_s = time.perf_counter() - tb
    del d_pairs
    n, m = g.num_vertices(), g.num_edges()

    stream = torch.cuda.Stream(dev)
    plen = g.partials_len(world)
    partials = torch.empty(2 * plen, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    b, e = shard_range(m, world, rank)

    def step():
        return sharded_step(g, partials, rank, world, stream)[0]

    for _ in range(args.warmup):
        X = step()
    torch.cuda.synchronize()

    phase_ms = np.zeros(5)
    launches = 0
    step_ms = []
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            s_ev = torch.cuda.Event(enable_timing=True)
            e_ev = torch.cuda.Event(enable_timing=True)
            s_ev.record(stream)
            X = step()
            e_ev.record(stream)
            e_ev.synchronize()
            step_ms.append(s_ev.elapsed_time(e_ev))
            ms, nl, work = g.last_stats()
            phase_ms += np.array(ms)
            launches += nl
        torch.cuda.synchronize()
        barrier()
    clocks = clk.summary()
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = m * args.steps / (total_ms / 1e3)
    phase_ms /= args.steps
    ms, nl, work = g.last_stats()

    # the passes run one after the other on the step's stream (gl_set_overlap
    # default 0: running the cycle pass concurrently measured slower), so the
    # per-phase CUDA-event times of the timed steps are each pass alone
    phase_serial = phase_ms.copy()

    # ---- roofline of the dominant kernel (per-launch algorithmic bytes / event time)
    names = ["cliques_triangles", "triangle_sums", "cycles", "epilogue"]
    bytes_alg = [float(w) for w in work]  # algorithmic bytes per phase
    dom = int(np.argmax(phase_serial[:4]))
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = bytes_alg[dom] / (phase_serial[dom] / 1e3) / 1e9 if phase_serial[dom] > 0 else 0.0
    # DRAM bytes of the dominant kernel from an ncu capture OF THIS WORKLOAD
    # (profiles/traffic.json, keyed by workload); null when none was taken
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            ent = json.load(open(tpath)).get("workloads", {}).get(workload_key(args), {})
            traffic, traffic_src = ent.get(names[dom]), ent.get("source")
        except Exception:
            traffic = None

    # ---- e2e through the public C-ABI from pinned host buffers.  The
    # device-resident graph is released first: every e2e graph is built, counted
    # and freed on its own (each count sizes its H-edge record list from the
    # free memory, so graphs alive side by side at RMAT-24+ would run out)
    g.close()
    del partials, flush
    torch.cuda.synchronize()
    e2e = None
    if not args.no_e2e:
        hpairs = hp if hp is not None else host_pairs(args)
        pin_in = torch.from_numpy(hpairs.view(np.int64).reshape(-1)).pin_memory()
        shard_n = e - b
        pin_t = torch.empty(max(1, shard_n), dtype=torch.int32).pin_memory()
        pin_x7 = torch.empty(max(1, shard_n), dtype=torch.int64).pin_memory()
        pin_x10 = torch.empty(max(1, shard_n), dtype=torch.int64).pin_memory()
        e2e_ms = []
        # second variant: the reference caller's full per-edge output, every
        # 80-byte MicroRecord (counts.hpp:82-89) of the shard, into pinned memory
        pin_rec = torch.empty(max(1, shard_n) * 80, dtype=torch.uint8).pin_memory()
        rec_view = pin_rec.numpy().view(gl.MICRO_DTYPE)[:shard_n]
        rec_ms = []
        for i in range(args.e2e_steps + args.e2e_warmup):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g2 = gl.Graph.build_host_ptr(pin_in.data_ptr(), count, local)  # gl_graph_build
            m2 = g2.num_edges()
            p2 = None
            if world == 1:
                # gl_count_edges: t and x7 leave the device while the cycle pass runs
                res2, _, _, _ = g2.count_edges(pin_t.numpy().view(np.uint32)[:shard_n],
                                               pin_x7.numpy().view(np.uint64)[:shard_n],
                                               pin_x10.numpy().view(np.uint64)[:shard_n])
                X2 = res2.X
            else:
                p2 = torch.empty(2 * g2.partials_len(world), dtype=torch.int64, device=dev)
                X2, _ = sharded_step(g2, p2, rank, world, stream)
                g2.edge_counts(b, shard_n, pin_t.numpy().view(np.uint32)[:shard_n],
                               pin_x7.numpy().view(np.uint64)[:shard_n], pin_x10.numpy().view(np.uint64)[:shard_n])
            dt = (time.perf_counter() - t0) * 1e3
            g2.close()
            del p2
            # same step again on a fresh graph, ending in the full MicroRecord
            # table instead of the compact (t, x7, x10) arrays
            barrier()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            g3 = gl.Graph.build_host_ptr(pin_in.data_ptr(), count, local)
            p3 = torch.empty(2 * g3.partials_len(world), dtype=torch.int64, device=dev)
            X3, _ = sharded_step(g3, p3, rank, world, stream)
            g3.micro_records(b, shard_n, out=rec_view)
            dr = (time.perf_counter() - t1) * 1e3
            if os.environ.get("GL_BENCH_VERBOSE"):
                print(f"e2e iteration {i}: {dt:.1f} ms, with micro records {dr:.1f} ms", file=sys.stderr, flush=True)
            g3.close()
            del p3
            if i >= args.e2e_warmup:  # warm-up iterations: first-touch allocations
                e2e_ms.append(dt)
                rec_ms.append(dr)
            assert X2 == X and X3 == X, "e2e counts differ from device-resident counts"
        tot, tot_rec = sum(e2e_ms), sum(rec_ms)
        if world > 1:
            t = torch.tensor([tot, tot_rec], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tot, tot_rec = (float(x) for x in t.tolist())
        e2e = {"value": m * len(e2e_ms) / (tot / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(pin_in.numel() * 8),
               "d2h_bytes_per_step": int(shard_n * (4 + 8 + 8) + 18 * 16),
               "ms_per_step": tot / max(1, len(e2e_ms)),
               "includes": "H2D of the raw label pairs, on-device CSR build, count, D2H of the COMPACT per-edge "
                           "output (t u32, x7 u64, x10 u64 = 20 B/edge; the other MicroRecord fields are "
                           "closed-form in t and the degrees, counts.cpp:113-136) + X; at one rank through "
                           "gl_count_edges, whose t/x7 copies run while the cycle pass computes",
               "micro_records": {
                   "value": m * len(rec_ms) / (tot_rec / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": int(pin_in.numel() * 8),
                   "d2h_bytes_per_step": int(shard_n * 80 + 18 * 16),
                   "ms_per_step": tot_rec / max(1, len(rec_ms)),
                   "includes": "same step ending in the full 80-byte MicroRecord table (micro_counts, "
                               "counts.cpp:122-136) of every edge, D2H into pinned memory"}}

    # ---- e2e from an edge-list TEXT (load_edge_list, graph.cpp:47-85): the
    # same step starting from the file bytes in pinned host memory, parsed on
    # the device (gl_graph_build_text) -- and, once, parsed by the host scanner
    # (gl_load_edge_list + gl_graph_build) for comparison.  World 1, m <= 2^25
    # (the text is formatted in Python once, outside the timed region).
    if e2e is not None and world == 1 and m <= (1 << 25) and not args.no_text_e2e:
        hp2 = hp if hp is not None else host_pairs(args)
        txt = ("\n".join(f"{a} {c}" for a, c in hp2.tolist()) + "\n").encode()
        pin_txt = torch.frombuffer(bytearray(txt), dtype=torch.uint8).pin_memory()
        tms = []
        for i in range(args.e2e_steps + args.e2e_warmup):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            g4 = gl.Graph.build_text((pin_txt.data_ptr(), pin_txt.numel()), local)  # gl_graph_build_text
            res4, _, _, _ = g4.count_edges(pin_t.numpy().view(np.uint32)[:m], pin_x7.numpy().view(np.uint64)[:m],
                                           pin_x10.numpy().view(np.uint64)[:m])
            X4 = res4.X
            dt = (time.perf_counter() - t0) * 1e3
            g4.close()
            assert X4 == X, "text e2e counts differ"
            if i >= args.e2e_warmup:
                tms.append(dt)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g5 = gl.Graph.build(gl.load_edge_list(txt), local)  # host scanner + gl_graph_build
        res5, _, _, _ = g5.count_edges(pin_t.numpy().view(np.uint32)[:m], pin_x7.numpy().view(np.uint64)[:m],
                                       pin_x10.numpy().view(np.uint64)[:m])
        X5 = res5.X
        host_ms = (time.perf_counter() - t0) * 1e3
        g5.close()
        assert X5 == X
        e2e["from_text"] = {
            "value": m * len(tms) / (sum(tms) / 1e3), "unit": UNIT, "h2d_bytes_per_step": len(txt),
            "d2h_bytes_per_step": int(m * (4 + 8 + 8) + 18 * 16), "ms_per_step": sum(tms) / len(tms),
            "includes": "H2D of the edge-list text (pinned), load_edge_list rules on the device (parse.cu), "
                        "CSR build, count, D2H of t/x7/x10 + X",
            "host_parser_ms_per_step": host_ms,
            "host_parser_note": "same step with the text parsed by the host scanner (gl_load_edge_list, one "
                                "thread) and the pairs copied from pageable memory; one step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        hpairs = hp if hp is not None else host_pairs(args)
        rates, cores, kind, desc = cpu_sample_run(hpairs, args.cpu_seconds)
        cpu = {"value": rates[0], "unit": UNIT, "cores": cores, "kind": kind, "sample": desc}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": ("synthetic (BA generated on the host, seed %d)" % args.seed if args.graph == "ba"
                     else "synthetic (RMAT generated on device, seed %d)" % args.seed),
            "config": dict(workload(args), n=n, m=m, parallelism=f"replicated graph, {world} rank work shares",
                           l2="flushed (256 MiB write) before every step, outside the timed events"),
            "e2e": e2e,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": names[dom], "achieved": achieved, "peak": peak,
                         "duration_ms": float(phase_serial[dom]),
                         "duration_source": "CUDA events around the pass on the launching stream, passes serialised "
                                            "(the default, gl_set_overlap(0)), averaged over the timed steps",
                         "unit": "GB/s", "frac": achieved / peak if peak else None, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": bytes_alg[dom],
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if peaks else "fallback 6650"},
            "phase_ms": {k: float(v) for k, v in zip(names + ["sum"], phase_ms)},
            "phase_ms_serial": {k: float(v) for k, v in zip(names + ["sum"], phase_serial)},
            "build_ms": build_s * 1e3,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "X": [str(x) for x in X],
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
