#!/usr/bin/env python3
"""GPops/s of the tree-evaluation hot path on B200 (BASELINE.json metric).

Workload (config.workload = "c3"): BASELINE.json configs[2] — the
evaluation-only batch of 4000 seeded random prefix trees, node counts
log-uniform in [10^4, 10^6] (~8.6e8 nodes, ~4.1e10 GPops), ops uniform over
{+,-,*,/}, leaves 50% x / 50% constants in [-1,1], 48 Sextic fitness cases.
It is the largest config that is a pure pass of the hot path over one batch;
configs[1] (pop 4000 evolution) is a parity case whose per-generation work is
microseconds.

One step = evaluate_population over the whole batch (per-case outputs, MAE
fitness, hits, size, depth of every tree). With --gpus N (torchrun, one
process per GPU) the population is N config-3 batches, one per rank (rank r
uses corpus seed SEED + r): weak scaling, fixed work per GPU. Every step ends
with an NCCL all-gather of the 16-byte per-individual records, so every rank
holds the whole population's fitness for tournament selection.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 1
M_TREES = 4000
LG_LO, LG_HI = 4.0, 6.0
LANES = 48
METRIC = "GPops/s (tree nodes x fitness cases evaluated per sec)"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 9:
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_info():
    """CPU model and hardware threads of this host (BASELINE.md's CPU plan)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "nproc": os.cpu_count() or 1}


def workload_config(world, sizes_of):
    """The config dict both arms print (identical keys and values): the
    config-3 batch per GPU, seeds SEED + r for r < world."""
    sizes = [sizes_of(SEED + r) for r in range(world)]
    nodes = sum(int(s.sum()) for s in sizes)
    return {"workload": "c3", "trees_per_gpu": M_TREES, "lg_nodes": [LG_LO, LG_HI],
            "seeds": [SEED + r for r in range(world)], "nodes": nodes, "gpops_per_step": nodes * LANES,
            "parallelism": f"population shards x{world}" + (" + NCCL all-gather of records" if world > 1 else ""),
            "l2": "inputs larger than L2: %.0f MB of opcodes per GPU vs 126 MB L2" % (int(sizes[0].sum()) / 1e6)}


def oracle_sample(threads, seconds_target, first_trees=None):
    """Time the oracle's multi-threaded evaluate_population (the reference's
    CPU algorithm as restated in oracle/) on a prefix of the workload. Only
    the oracle library is loaded here: suite and corpus come from its own
    generators (byte-identical to the product's, tests/test_oracle.py)."""
    from tests._oracle import load_oracle

    o = load_oracle()
    suite = o.make_suite(int(o.orc_suite_seed(SEED)))
    sizes = o.corpus_sizes(SEED, M_TREES, LG_LO, LG_HI)
    # calibrate on the first few trees
    n_cal = 8
    buf, offs, sz = o.corpus(SEED, M_TREES, LG_LO, LG_HI, first=0, n=n_cal)
    t0 = time.perf_counter()
    o.evaluate_population(buf, offs, sz, suite, threads=threads)
    rate = float(sz.sum()) / max(time.perf_counter() - t0, 1e-6)  # nodes/s
    budget = rate * seconds_target
    if first_trees is None:
        csum = np.cumsum(sizes.astype(np.float64))
        first_trees = int(min(M_TREES, max(n_cal, np.searchsorted(csum, budget) + 1)))
    buf, offs, sz = o.corpus(SEED, M_TREES, LG_LO, LG_HI, first=0, n=first_trees)
    return o, suite, buf, offs, sz, first_trees


def run_reference(args, rank, world):
    """The reference's CPU path (the oracle port: the reference is a header
    skeleton without function bodies, so its own evaluator cannot be built)
    on all host threads, rank 0 only. Never loads the product libraries."""
    if rank != 0:
        return
    from tests._oracle import load_oracle

    threads = os.cpu_count() or 1
    per_step = max(2.0, min(10.0, 150.0 / max(1, args.steps + args.warmup)))
    o, suite, buf, offs, sz, ntrees = oracle_sample(threads, per_step)
    nodes = int(sz.sum())
    for _ in range(args.warmup):
        o.evaluate_population(buf, offs, sz, suite, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.evaluate_population(buf, offs, sz, suite, threads=threads)
    dt = time.perf_counter() - t0
    value = nodes * LANES * args.steps / dt
    cpu = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GPops/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded config-3 corpus, generated on the host)",
        "config": workload_config(world, lambda sd: o.corpus_sizes(sd, M_TREES, LG_LO, LG_HI)),
        "cpu_baseline": {"value": value, "unit": "GPops/s", "cores": threads, "kind": "port",
                         "cpu": cpu,
                         "sample": f"first {ntrees} of {M_TREES} config-3 trees ({nodes} nodes) per step; "
                                   f"oracle eval_batch (48-lane AVX frames, the reference's eval_batch_raw "
                                   f"restated) on a {threads}-thread dynamic pool; the reference itself is "
                                   f"declarations only and cannot run"},
        "e2e": {"value": value, "unit": "GPops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1902_09215_b200 as ltgp

    torch.cuda.set_device(local_rank)
    pk, pk_kind = peaks()
    # weak scaling: rank r owns population slots [r*M, (r+1)*M), a config-3
    # batch generated from corpus seed SEED + r
    ranges = [(r * M_TREES, M_TREES) for r in range(world)]
    first, count = 0, M_TREES
    nodes_job = sum(int(ltgp.corpus_sizes(SEED + r, M_TREES, LG_LO, LG_HI).sum()) for r in range(world))
    bytes_job = sum(int(((ltgp.corpus_sizes(SEED + r, M_TREES, LG_LO, LG_HI) + 15) // 16 * 16).sum())
                    for r in range(world))
    pinned_keep = []

    def pinned(nbytes):
        t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        pinned_keep.append(t)
        return t.numpy()

    buf, offs, sizes = ltgp.corpus(SEED + rank, M_TREES, LG_LO, LG_HI, pinned=pinned, first=first, n=count)
    nodes_rank = int(sizes.sum())
    suite = ltgp.make_suite(ltgp.suite_seed(SEED))
    e = ltgp.Engine([local_rank], node_limit=15_000_000)
    e.set_suite(*suite)
    e.upload_packed(buf, offs, sizes)
    rec = np.zeros(count, ltgp.RECORD_DTYPE)
    dptr, _, _, sptr = e.shard_records(0)
    estream = torch.cuda.ExternalStream(sptr)
    if world > 1:
        # the engine joins the ranks' NCCL communicator (ltgp_nccl_attach):
        # every evaluation then all-gathers the ranks' records inside the
        # engine (one ncclAllGather over NVLink; the tournament-selection
        # exchange), the same code the run loop's record gather uses
        uid = [ltgp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        e.nccl_attach(uid[0], world, rank)

    def gather():
        pass  # inside evaluate_collect / evaluate_packed (the engine's all-gather)

    def step(host_records=True):
        e.evaluate_launch()
        e.evaluate_collect(rec if host_records else None)
        gather()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(args.warmup, 3) if args.warmup >= 0 else 3):
        step()
    # ---------------- device-resident throughput (value) ----------------
    clocks = ClockSampler(local_rank)
    clocks.start()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(estream)
    kern = []
    comb = []
    launches = 0
    for _ in range(args.steps):
        step()
        st = e.stats()
        kern.append(st["keval_seconds"])  # k_eval alone (CUDA events around its launch)
        comb.append(st["combine_seconds"])
        launches += st["kernel_launches"]
    ev1.record(torch.cuda.current_stream())
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    t_max = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())
    value = nodes_job * LANES * args.steps / (ms * 1e-3)
    kern_s = float(np.mean(kern))
    # ---------------- end to end through the C ABI (e2e) ----------------
    barrier()
    ev2 = torch.cuda.Event(enable_timing=True)
    ev3 = torch.cuda.Event(enable_timing=True)
    e.evaluate_packed(buf, offs, sizes, rec=rec)  # warm the streamed path's work-list cache
    barrier()
    ev2.record(estream)
    for _ in range(args.steps):
        # one reference-facing call per step: H2D of the step's trees from
        # pinned memory (in slices, overlapped with their evaluation) and
        # D2H of the records
        e.evaluate_packed(buf, offs, sizes, rec=rec)
        gather()
    ev3.record(torch.cuda.current_stream())
    barrier()
    ms_e2e = ev2.elapsed_time(ev3)
    t_e2e = torch.tensor([ms_e2e], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    ms_e2e = float(t_e2e.item())
    e2e = nodes_job * LANES * args.steps / (ms_e2e * 1e-3)
    # bytes that crossed PCIe per step: the packed slices (ltgp_pack.h)
    h2d = torch.tensor([float(e.stats()["last_h2d_bytes"])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(h2d, op=dist.ReduceOp.SUM)
    h2d_job = int(h2d.item())
    # ---------------- roofline of the dominant kernel (k_eval) ----------------
    sms = torch.cuda.get_device_properties(local_rank).multi_processor_count
    peak_tops = sms * 128 * pk["sm_max_mhz"] * 1e6 / 1e12  # FP32 lanes/clk x clock, 1 GPop = 1 op
    achieved = nodes_rank * LANES / kern_s / 1e12
    traffic = None
    binding = None
    prof = os.path.join(ROOT, "profiles", "ncu_k_eval.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            traffic = pj.get("dram_bytes_per_launch")
            mp = pj.get("metrics_pct", {})
            # what actually bounds the interpreter: the
            # per-pair dependent chain (indirect branch, operand loads) and
            # issue slots, not the FP32 pipe or HBM
            binding = {
                "resource": "latency of each warp's per-pair chain at 32 resident warps: with the direct-threaded "
                            "dispatch the stall samples (profiles/r02c_keval_stalls.txt) are branch resolution "
                            "after the handler's BRX 22% (+9% instruction fetch at its target), shared-memory "
                            "scoreboard 20%, fixed-latency dependencies 18%; issue slots ~70% busy; the "
                            "shared-memory pipe (83%) does not bind yet (broadcast-leaf probe, DESIGN.md 3.9)",
                "issue_active_pct": float(mp.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "nan")),
                "shared_wavefronts_pct": float(mp.get(
                    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "nan")),
                "fma_pipe_pct": float(mp.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "nan")),
                "inst_per_node": pj.get("instructions_per_node"),
                "shared_wavefronts_per_node": pj.get("shared_wavefronts_per_node"),
                "source": "profiles/ncu_k_eval.json (ncu --set full of the same k_eval on this workload)"}
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "GPops/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded config-3 corpus, generated on the host)",
        "config": workload_config(world, lambda sd: ltgp.corpus_sizes(sd, M_TREES, LG_LO, LG_HI)),
        "e2e": {"value": e2e, "unit": "GPops/s", "h2d_bytes_per_step": h2d_job, "opcode_bytes_per_step": bytes_job,
                "transfer": "each ~18 MB slice of the caller's pinned buffer is packed by the host threads inside "
                            "the timed call (3-bit codes, constants as literal bytes; csrc/ltgp_pack.h) and sent; "
                            "one persistent k_eval rebuilds, decodes, plans and evaluates every slice as it lands "
                            "(cross-slice task queue, the copy stream marks each slice with a stream memory op)",
                "d2h_bytes_per_step": M_TREES * 16 * world},
        "gpu_launches": launches,
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak_tops, "unit": "TFLOP/s",
                     "frac": achieved / peak_tops, "traffic": traffic,
                     "note": f"k_eval only (CUDA events around its launch on the engine stream): {nodes_rank} "
                             f"nodes x 48 ops / {kern_s * 1e3:.3f} ms avg launch; "
                             f"peak = {sms} SMs x 128 FP32 lanes x {pk['sm_max_mhz']:.0f} MHz ({pk_kind} clock); "
                             f"opcode stream {nodes_rank / kern_s / 1e9:.1f} GB/s of {pk['hbm_gbs']:.0f} GB/s HBM ({pk_kind})",
                     "combine_ms": float(np.mean(comb)) * 1e3, "binding": binding},
        "clocks": clk,
    }
    if world > 1:
        g = e.gathered_records()
        ok = g.size == world * count and g[rank * count:(rank + 1) * count].tobytes() == rec.tobytes()
        line["collective"] = {"impl": e.gather_mode(), "op": "ncclAllGather of the 16-byte records every step",
                              "nranks": world, "gather_ms": e.stats()["gather_seconds"] * 1e3,
                              "own_block_matches": bool(ok)}
    if world == 1 and rank == 0 and not args.no_evolution:
        # secondary: BASELINE configs[1] (pop 4000, k=7, crossover only, no size
        # limit, 200 generations, bloating 50/50-grow variant — see DESIGN.md
        # §6), run by the C++ host loop with splice + evaluation on the device
        e.close()
        with ltgp.Engine([local_rank], node_limit=2**62) as ev:
            # warm-up run: the engine's device and pinned buffers grow to the
            # run's sizes once (first-run wall times varied 0.25-0.6 s)
            ev.run(4000, 200, 2**62, 7, SEED, None, 1)
            t0 = time.perf_counter()
            r = ev.run(4000, 200, 2**62, 7, SEED, None, 1)
            wall = time.perf_counter() - t0
        line["evolution_c2"] = {
            "generations": r["generations"], "nodes": r["nodes"],
            "eval_gpops_per_s": r["nodes"] * LANES / max(r["eval_seconds"], 1e-12),
            "e2e_gpops_per_s": r["nodes"] * LANES / wall, "wall_s": wall,
            "note": "per-generation device evaluation (splice excluded) and whole-run wall clock incl. host planning"}
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        o, s2, cb, co, cs, ntrees = oracle_sample(threads, args.cpu_seconds)
        t0 = time.perf_counter()
        o.evaluate_population(cb, co, cs, s2, threads=threads)
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": float(cs.sum()) * LANES / dt, "unit": "GPops/s", "cores": threads,
                                "kind": "port", "cpu": cpu_info(),
                                "sample": f"first {ntrees} of {M_TREES} config-3 trees ({int(cs.sum())} nodes); "
                                          f"oracle eval_batch on a {threads}-thread pool, {dt:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    e.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-evolution", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
