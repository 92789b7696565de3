#!/usr/bin/env python
"""Benchmark: GF(2)[x] multiply at the paper's headline sizes (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4b|c4a|c3|c2|c1] [--impl ours|reference]

A "step" is one whole Alg. 5 multiply (every §8(a) row: Split, BasisCvt, changeRepr, FFT_LCH x2,
pointmul, iFFT_LCH, iBasisCvt, changeRepr^-1, InterleavedCombine) of two seeded uniformly random
operands (gf2x_synth recipe) already resident in HBM.  Time = CUDA events on the library's stream
around exactly K steps after W warm-ups, barrier + synchronize on both sides, max over ranks.
value = input Gbit/s = (a_bits + b_bits) * steps * n_gpus / max-rank time (whole job).

Multi-GPU (torchrun, N > 1): by default ONE multiply partitioned over the N ranks (SURVEY §8(e):
gf2x_mul_sharded, NCCL all-gather + all-to-all/pairwise exchanges, top log2 N FFT layers as the
exchange step; "scaling": "strong"; value = input bits of that multiply / max-rank time); rank 0
checks the gathered product against its own single-GPU multiply.  --mode replicas runs one
independent multiply per rank instead ("scaling": "weak"); batched configs always shard that way.

--impl reference runs the repo's CPU oracle (oracle/, the paper's Alg. 5 step by step) on the box's
host cores on a bounded sample of the same workload (rank 0 only) and prints the same JSON line.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from gf2x_synth import CONFIGS, DEFAULT_SEED, batch_pair, operand_pair  # noqa: E402

METRIC = "ms per 2^28- and 2^29-bit GF(2)[x] multiply; input Gbit/s; % of HBM roofline"
UNIT = "input Gbit/s"
PAPER_GBITS = {"c4a": (2 * 2**28) / 2.302 / 1e9, "c4b": (2 * 2**29) / 4.812 / 1e9, "c3": (2 * 2**24) / 0.104 / 1e9}
PAPER_MS = {"c4a": 2302.0, "c4b": 4812.0, "c3": 104.0}
WORKLOAD = {
    "c1": "single 2^16-bit x 2^16-bit GF(2)[x] multiply (FFT over 2^11 TGF(2^128) points)",
    "c2": "4096 independent 2^14-bit x 2^14-bit multiplies (batched, 2^9 points each)",
    "c3": "single 2^24-bit x 2^24-bit multiply (2^19 points)",
    "c4a": "single 2^28-bit x 2^28-bit multiply (2^23 points), paper headline size",
    "c4b": "single 2^29-bit x 2^29-bit multiply (2^24 points), paper headline size",
    "c5": "single 2^32-bit x 2^32-bit multiply (2^27 points), 2^33-bit product",
}


def rank_info():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_alu_peak():
    """ALU-pipe peak in lane instructions/s: 148 SMs x 4 SMSPs x 16 lanes/clk (LOP3/PRMT/SHF issue every 2nd
    cycle per SMSP, B300_MICROARCH.md "Pipe rates") x the max SM clock (MEASURED_PEAKS.json sm_max_mhz, else
    the 1965 MHz of B200_PROFILING.md)."""
    mhz, src = 1965.0, "derived: 148 SM x 64 lanes/clk x 1965 MHz (B200_PROFILING.md clocks.max.sm)"
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            mhz = float(json.load(open(p))["sm_max_mhz"])
            src = f"derived: 148 SM x 64 lanes/clk x {mhz:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)"
        except Exception:
            pass
    return 148 * 64 * mhz * 1e6 / 1e9, src


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append((time.time(), ln.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        sm, mx, reasons = [], None, set()
        for ts, ln in self.lines:
            if ts < t0 or ts > t1:
                continue
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(cfg: str, bits: int, batch: int, alg=5):
    """The oracle as it stands (plain C, OpenMP; the paper's Alg. 5 step by step, or App. C for --alg frob),
    timed on this box's host cores (SURVEY §8(d) / BASELINE.md §3):
      * O3 on the benched workload itself at all host cores (one run; for batched configs a bounded sample
        of 64 of the pairs);
      * O3 at 1 thread, median of 3, on a stated 2^22-bit size (the paper's single-core setting);
      * O2 Karatsuba at 1 thread on 2^24-bit operands (where it finishes).
    `value` is the all-cores figure on the benched workload."""
    import oracle as O
    O.build()
    allc = O.num_threads()
    fn, name = (O.frob_mul, "App. C (Frobenius bijection)") if alg == "frob" else (O.alg5_mul, "Alg. 5")
    if batch == 1:
        a, b = operand_pair(bits, DEFAULT_SEED)
        t0 = time.perf_counter()
        fn(a, bits, b, bits)
        dt_all = time.perf_counter() - t0
        all_bits, all_what = 2 * bits, f"one multiply of the benched workload ({cfg}, 2 x {bits} bits)"
    else:
        k = min(batch, 64)
        A, B = batch_pair(bits, batch, DEFAULT_SEED)
        t0 = time.perf_counter()
        for i in range(k):
            fn(A[i], bits, B[i], bits)
        dt_all = time.perf_counter() - t0
        all_bits, all_what = 2 * bits * k, f"{k} of the {batch} pairs of {cfg} (2 x {bits} bits each)"
    val = 2 * all_bits / 2 / dt_all / 1e9
    # 1 thread, median of 3 (the paper's Table 2 runs are single-core: P:1184-1191)
    one_bits = min(bits, 1 << 22)
    a1, b1 = operand_pair(one_bits, DEFAULT_SEED)
    O.set_threads(1)
    try:
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            fn(a1, one_bits, b1, one_bits)
            ts.append(time.perf_counter() - t0)
        t1 = statistics.median(ts)
        kb = None
        if alg != "frob":
            kbits = min(bits, 1 << 24)
            ak, bk = operand_pair(kbits, DEFAULT_SEED)
            t0 = time.perf_counter()
            O.mul_karatsuba(ak, bk)
            kb = {"bits": kbits, "ms": round((time.perf_counter() - t0) * 1e3, 1),
                  "value": round(2 * kbits / (time.perf_counter() - t0) / 1e9, 6)}
    finally:
        O.set_threads(allc)
    return {"value": round(val, 6), "unit": UNIT, "cores": allc, "kind": "oracle",
            "sample": f"oracle {name} (O3) at all {allc} host threads: {all_what}, {dt_all * 1e3:.1f} ms",
            "nproc": os.cpu_count(), "cpu_model": _cpu_model(), "clmul": O.clmul_impl(),
            "one_thread": {"bits": one_bits, "ms_median_of_3": round(t1 * 1e3, 2),
                           "value": round(2 * one_bits / t1 / 1e9, 6), "kind": f"oracle {name} (O3), 1 thread"},
            "karatsuba_one_thread": kb}


REF_SAMPLE_BITS = 1 << 24   # the paper's Table 2 column 18 size (c3)


def run_reference(args):
    """The reference arm: the repo's CPU oracle (the paper's Alg. 5 step by step) on the host cores, each step one
    multiply of a bounded sample (two 2^24-bit operands) of the benched workload; rank 0 only."""
    rank, world, _ = rank_info()
    if rank != 0:
        return 0
    import oracle as O
    O.build()
    bits, _ = CONFIGS[args.config]
    sample_bits = min(bits, REF_SAMPLE_BITS)
    a, b = operand_pair(sample_bits, DEFAULT_SEED)
    for _ in range(args.warmup):
        O.alg5_mul(a, sample_bits, b, sample_bits)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.alg5_mul(a, sample_bits, b, sample_bits)
    dt = time.perf_counter() - t0
    val = 2 * sample_bits * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3 / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "config": args.config},
        "cpu_baseline": {"value": round(val, 6), "unit": UNIT, "cores": O.num_threads(), "kind": "oracle",
                         "sample": f"each step: one oracle Alg. 5 multiply of two 2^{sample_bits.bit_length() - 1}-bit "
                                   f"operands (bounded sample of {args.config}, same seeded recipe)",
                         "nproc": os.cpu_count(), "cpu_model": _cpu_model(), "clmul": O.clmul_impl()},
        "e2e": {"value": round(val, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def load_traffic(cfg):
    """ncu DRAM bytes per launch (by bench kernel name) and per whole multiply, from profiles/ncu_traffic.json."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(tpath)).get(cfg, {})
    except Exception:
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4b", choices=["c1", "c2", "c3", "c4a", "c4b", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--graph", action="store_true",
                    help="time replays of one step captured in a CUDA graph (launch overhead removed; for the small configs)")
    ap.add_argument("--bits", type=int, default=None,
                    help="operand size override: one multiply of two BITS-bit operands instead of --config's "
                         "(e.g. 268435520 = 2^28 + 64, the truncated-FFT staircase, DESIGN.md §10c)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-companion", action="store_true",
                    help="c4b: do not also time the 2^28-bit multiply (c4a) in the same run")
    ap.add_argument("--w", type=int, default=64, choices=[64, 128],
                    help="Alg. 5 block width: 64 (TGF(2^128), default) or 128 (TGF(2^256), P:873-874)")
    ap.add_argument("--alg", default="5", choices=["5", "4", "frob"],
                    help="5: Alg. 5 over the tower (default); 4: Alg. 4 in GF(2^128) polynomial basis (P:562-614); "
                         "frob: App. C, the Frobenius bijection (P:1485-1552; one product per step)")
    ap.add_argument("--mode", default=None, choices=["sharded", "replicas"],
                    help="N > 1: one multiply partitioned over the ranks (default) or one per rank")
    args = ap.parse_args()
    args.alg = int(args.alg) if args.alg.isdigit() else args.alg
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1708_09746_b200 as G

    rank, world, local = rank_info()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    G.load()
    bits, batch = CONFIGS[args.config]
    if args.bits:
        bits, batch = args.bits, 1
        args.config = "custom"
        plan = G.gf2x_plan(bits, bits)
        WORKLOAD["custom"] = (f"single {bits}-bit x {bits}-bit multiply ({plan['N']} points"
                              + (f", truncated FFT: H-point + 2^{plan['trunc_j']}-point multiplies" if plan["trunc_j"] >= 0 else "")
                              + (", split BasisCvt" if any(plan["split"].values()) else "") + ")")
        if args.mode is None and world > 1:
            args.mode = "replicas"
    if args.alg == "frob" and (batch != 1 or args.w != 64):
        print("[bench] --alg frob runs one product of 64-bit-word operands per step (no batch, w = 64)", file=sys.stderr)
        return 2
    mode = args.mode or ("sharded" if world > 1 else "single")
    if world == 1:
        mode = "single"
    if mode == "sharded" and (batch != 1 or args.w != 64 or args.alg != 5):
        mode = "replicas"   # batched configs shard trivially: independent products per rank
    sharded = mode == "sharded"
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    def operands(nbits, nbatch, seed):
        if nbatch == 1:
            x, y = operand_pair(nbits, seed)
        else:
            x, y = batch_pair(nbits, nbatch, seed)
        dx = torch.from_numpy(x.reshape(-1).view(np.int64)).to(dev).view(torch.uint64)
        dy = torch.from_numpy(y.reshape(-1).view(np.int64)).to(dev).view(torch.uint64)
        return x, y, dx, dy

    seed = DEFAULT_SEED + (0 if sharded else 2 * rank)  # replicas: each rank its own operand pair
    a, b, da, db = operands(bits, batch, seed)
    n = G.nwords(bits)
    n_out = 2 * n
    dc = torch.empty(n_out * batch, dtype=torch.uint64, device=dev)

    def fail_line(err):
        """A failed partitioned multiply prints a line that carries no throughput (never a replicas number)."""
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                              "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                              "scaling": "failed", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                              "config": {"workload": WORKLOAD[args.config], "config": args.config,
                                         "parallelism": f"sharded FFT over {world} GPUs"},
                              "sharded_error": err, "gpu_launches": 0}), flush=True)
        if dist:
            dist.destroy_process_group()
        return 1

    if sharded:
        # the FFT partitioned over the ranks (NCCL over NVLink); rank r owns words
        # [r n/G, (r+1) n/G) of a and b and receives words [r 2n/G, (r+1) 2n/G) of c
        err = None
        try:
            comm = G.init_from_process_group()
            lo, hi = G.shard_words(n, world, rank)
            sa, sb = da[lo:hi].clone(), db[lo:hi].clone()
            sc = torch.empty(n_out // world, dtype=torch.uint64, device=dev)
            comm.mul(sa, sb, bits, sc, stream=stream)
            comm.wait(stream, timeout_s=300.0)   # NCCL async errors / a dead peer abort instead of hanging
            ok = 1
        except Exception as e:   # e.g. NCCL unavailable: every rank sees it (same library, same lists)
            err, ok = f"{type(e).__name__}: {e}"[:300], 0
        flag = torch.tensor([ok], dtype=torch.int32, device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 1:
            # the first partitioned product must equal the single-GPU one (rank 0 checks)
            parts = [torch.empty_like(sc) for _ in range(world)]
            dist.all_gather(parts, sc)
            if rank == 0:
                G.gf2x_mul(da, bits, db, bits, dc, stream=stream)
                torch.cuda.synchronize()
                if not torch.equal(torch.cat(parts).view(torch.int64), dc.view(torch.int64)):
                    ok, err = 0, "sharded product differs from the single-GPU product"
            flag = torch.tensor([ok], dtype=torch.int32, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            return fail_line(err or "another rank failed")

    def make_step(xa, xb, xc, nbits, nbatch):
        def step():
            if sharded:
                comm.mul(sa, sb, bits, sc, stream=stream)
            elif args.alg == "frob":
                G.gf2x_mul_frob(xa, nbits, xb, nbits, xc, stream=stream)
            elif args.alg == 4:
                G.gf2x_mul_alg4(xa, nbits, xb, nbits, nbatch, xc, stream=stream)
            elif args.w != 64:
                G.gf2x_mul_w(xa, nbits, xb, nbits, args.w, nbatch, xc, stream=stream)
            elif nbatch == 1:
                G.gf2x_mul(xa, nbits, xb, nbits, xc, stream=stream)
            else:
                G.gf2x_mul_batched(xa, nbits, xb, nbits, nbatch, xc, stream=stream)
        return step

    step = make_step(da, db, dc, bits, batch)

    def timed(fn, steps):
        """W warm-ups, then exactly `steps` calls bracketed by barrier + synchronize, CUDA events on the
        library stream; max over ranks.  No profiling hooks inside the timed region."""
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        tw0 = time.time()
        ev0.record(stream)
        for _ in range(steps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        tw1 = time.time()
        if dist:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        if dist:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, tw0, tw1

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ms, t_wall0, t_wall1 = timed(step, args.steps)
    ms_eager = None
    if args.graph and not sharded:
        # one step captured on a side stream (the library plans on the host at capture time), replayed K times
        ms_eager = ms
        eager_stream, stream = stream, torch.cuda.Stream()
        with torch.cuda.stream(stream):
            for _ in range(2):
                step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
        with torch.cuda.stream(stream):
            ms, t_wall0, t_wall1 = timed(graph.replay, args.steps)
        stream = eager_stream
    time.sleep(0.25)
    sampler.stop()
    clocks = sampler.summary(t_wall0 - 0.05, t_wall1 + 0.05)

    ms_step = ms / args.steps
    in_bits = 2 * bits * batch
    jobs = 1 if sharded else world   # multiplies the whole job completes per step
    value = in_bits * jobs / (ms_step * 1e-3) / 1e9
    if sharded:
        # the partitioned product equals the single-GPU one (rank 0 recomputes it alone)
        comm.check()
        parts = [torch.empty_like(sc) for _ in range(world)]
        dist.all_gather(parts, sc)
        if rank == 0:
            G.gf2x_mul(da, bits, db, bits, dc, stream=stream)
            torch.cuda.synchronize()
            assert torch.equal(torch.cat(parts).view(torch.int64), dc.view(torch.int64)), "sharded != single-GPU"

    # ---- per-kernel breakdown: a separate profiled run (CUDA events around every launch), not the headline
    nprof = max(1, min(args.steps, 10))
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    G.profile_enable(True)
    for _ in range(nprof):
        step()
    torch.cuda.synchronize()
    prof = G.profile_report()
    G.profile_enable(False)

    # ---- the 2^28-bit companion (BASELINE metric names both headline sizes): same protocol, same run
    companion = None
    if (args.config == "c4b" and not args.no_companion and not sharded and world == 1 and args.alg == 5
            and args.w == 64):
        cb, _ = CONFIGS["c4a"]
        _, _, ca, cbb = operands(cb, 1, DEFAULT_SEED)
        cc = torch.empty(2 * G.nwords(cb), dtype=torch.uint64, device=dev)
        cms, _, _ = timed(make_step(ca, cbb, cc, cb, 1), args.steps)
        cstep = cms / args.steps
        companion = {"config": "c4a", "workload": WORKLOAD["c4a"], "operand_bits": cb, "ms_per_step": round(cstep, 4),
                     "value": round(2 * cb / (cstep * 1e-3) / 1e9, 4), "unit": UNIT, "steps": args.steps,
                     "paper_ms_haswell": PAPER_MS["c4a"], "gpu_launches": G.gf2x_launch_count(cb, cb, 1) * args.steps}
        del ca, cbb, cc

    # ---- end to end through the public API with pinned host buffers.  Every step copies its operands
    # host -> device, multiplies, and copies the product device -> host; consecutive steps are pipelined
    # (H2D and D2H on their own streams / copy engines, two device buffer sets), as a user streaming
    # multiplies would run them.  Timed from the first H2D to the last D2H with CUDA events.
    if sharded:   # each rank moves its own shards
        ha = torch.from_numpy(a.reshape(-1)[lo:hi].view(np.int64)).pin_memory()
        hb = torch.from_numpy(b.reshape(-1)[lo:hi].view(np.int64)).pin_memory()
        n_c = n_out // world
    else:
        ha = torch.from_numpy(a.reshape(-1).view(np.int64)).pin_memory()
        hb = torch.from_numpy(b.reshape(-1).view(np.int64)).pin_memory()
        n_c = n_out * batch
    HC = [torch.empty(n_c, dtype=torch.int64).pin_memory() for _ in range(2)]
    EA = [torch.empty(ha.numel(), dtype=torch.int64, device=dev) for _ in range(2)]
    EB = [torch.empty(hb.numel(), dtype=torch.int64, device=dev) for _ in range(2)]
    EC = [torch.empty(n_c, dtype=torch.int64, device=dev) for _ in range(2)]
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def e2e_step(i):
        k = i & 1
        h2d_s.wait_event(ev_comp[k])           # step i-2's multiply has consumed EA[k], EB[k]
        with torch.cuda.stream(h2d_s):
            EA[k].copy_(ha, non_blocking=True)
            EB[k].copy_(hb, non_blocking=True)
        ev_in[k].record(h2d_s)
        stream.wait_event(ev_in[k])
        stream.wait_event(ev_out[k])           # step i-2's product has left EC[k]
        if sharded:
            comm.mul(EA[k], EB[k], bits, EC[k], stream=stream)
        elif args.alg == "frob":
            G.gf2x_mul_frob(EA[k], bits, EB[k], bits, EC[k], stream=stream)
        elif args.alg == 4:
            G.gf2x_mul_alg4(EA[k], bits, EB[k], bits, batch, EC[k], stream=stream)
        elif args.w != 64:
            G.gf2x_mul_w(EA[k], bits, EB[k], bits, args.w, batch, EC[k], stream=stream)
        elif batch == 1:
            G.gf2x_mul(EA[k], bits, EB[k], bits, EC[k], stream=stream)
        else:
            G.gf2x_mul_batched(EA[k], bits, EB[k], bits, batch, EC[k], stream=stream)
        ev_comp[k].record(stream)
        d2h_s.wait_event(ev_comp[k])
        with torch.cuda.stream(d2h_s):
            HC[k].copy_(EC[k], non_blocking=True)
        ev_out[k].record(d2h_s)

    for i in range(2):
        e2e_step(i)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(h2d_s)
    for i in range(args.e2e_steps):
        e2e_step(i)
    e1.record(d2h_s)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_val = in_bits * jobs / (e2e_ms / args.e2e_steps * 1e-3) / 1e9
    # result check of the e2e copies against the device-resident run (both from the library)
    ref = (sc if sharded else dc).cpu().view(torch.int64)
    assert all(torch.equal(h.view(torch.int64), ref) for h in HC)
    ha_bytes, hb_bytes, hc_bytes = ha.numel() * 8, hb.numel() * 8, n_c * 8

    # ---- roofline of the dominant kernel (CUDA-event durations of the profiled run) and the §8(d) fractions
    peak, peak_src = load_peaks()
    alu_peak, alu_src = load_alu_peak()
    dom = max(prof, key=lambda r: r["ms"])
    per_launch_ms = dom["ms"] / dom["launches"]
    per_launch_bytes = dom["bytes"] / dom["launches"]
    per_launch_ops = dom.get("alu_ops", 0) / dom["launches"]
    achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
    achieved_ops = per_launch_ops / (per_launch_ms * 1e-3) / 1e9
    tr = load_traffic(args.config)
    traffic = tr.get(dom["kernel"])
    step_bytes = sum(r["bytes"] for r in prof) / nprof
    kern_ms = sum(r["ms"] for r in prof) / nprof
    launches = G.gf2x_launch_count_w(bits, bits, batch, args.w)
    if sharded or args.alg in (4, "frob"):   # every kernel of these paths is bracketed by the profiling hook
        launches = sum(r["launches"] for r in prof) // nprof
    t_s = ms_step * 1e-3
    b_min = 32.0 * n * batch                       # read both operands once, write the product once
    b_ref = 320.0 * n * batch                      # SURVEY §8(d) 5-pass reference schedule (40 n W)
    ncu_step = tr.get("__step_dram_bytes")
    fractions = {
        "of": f"HBM {peak} GB/s ({peak_src}), whole multiply (ms_per_step)",
        "ncu_dram_bytes_per_multiply": ncu_step,
        "ncu_dram_frac": round(ncu_step / t_s / 1e9 / peak, 4) if ncu_step else None,
        "b_ref_bytes": b_ref, "b_ref_frac": round(b_ref / t_s / 1e9 / peak, 4),
        "b_min_bytes": b_min, "b_min_frac": round(b_min / t_s / 1e9 / peak, 5),
        "algorithmic_bytes_per_multiply": step_bytes,
        "algorithmic_frac": round(step_bytes / t_s / 1e9 / peak, 4),
    }
    kcommon = {"kernel": dom["kernel"], "launches_per_step": dom["launches"] / nprof,
               "algorithmic_bytes_per_launch": per_launch_bytes, "ms_per_launch": round(per_launch_ms, 5),
               "traffic_source": "profiles/ncu_traffic.json (ncu --set full, dram__bytes_read.sum + "
                                 "dram__bytes_write.sum per launch)" if traffic else None}
    if per_launch_ops > 0:
        roof = {"bound": "alu", "achieved": round(achieved_ops, 1), "peak": round(alu_peak, 1),
                "unit": "Ginstr/s (ALU-pipe lane instructions)", "frac": round(achieved_ops / alu_peak, 4),
                "traffic": traffic, "peak_source": alu_src,
                "frac_meaning": "issue fraction of the implementation's own instruction count: the kernel's designed "
                                "ALU-pipe instructions (SASS-counted, per launch) / its duration / the ALU-pipe peak",
                "algorithmic_alu_ops_per_launch": per_launch_ops,
                "hbm_achieved_gbs": round(achieved, 2), "hbm_frac": round(achieved / peak, 4), "hbm_peak": peak}
    else:
        roof = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src}
    roof.update(kcommon)
    roof["step"] = fractions

    line = {
        "metric": METRIC,
        "value": round(value, 4),
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": round(value / (PAPER_GBITS[args.config] * jobs), 2) if args.config in PAPER_GBITS else None,
        "vs_baseline_note": "ratio to the paper's own CPU number for this workload (Table 2, Haswell E3-1245 v3, "
                            "TGF(2^128) row): context, not the target",
        "dtype": "u64",
        "data": "synthetic",
        "config": {
            "workload": WORKLOAD[args.config] + ("" if args.w == 64 else ", w=128 blocks over TGF(2^256)")
                        + ("" if args.alg == 5 else (", Alg. 4 (GF(2^128) polynomial basis, dense multipliers)" if args.alg == 4
                           else ", App. C multiply through the Frobenius bijection (no Kronecker segmentation)")),
            "config": args.config, "operand_bits": bits, "batch": batch, "block_width": args.w, "algorithm": args.alg,
            "fft_points": 1 << max(0, (2 * n - 2).bit_length()) >> (0 if args.w == 64 else 1),
            **({"trunc_j": G.gf2x_plan(bits, bits)["trunc_j"]} if args.config == "custom" else {}),
            "parallelism": (f"sharded FFT over {world} GPUs (" + ("peer memory: CUDA IPC over NVLink, fused pull-pack "
                            "all-to-all, NCCL barriers" if comm.peer_memory() == 1 else "NCCL send/recv") + ")" if sharded else
                            ("replicas" if world > 1 else "single")),
            "seed": DEFAULT_SEED, "l2": "working set > 126 MB L2 (operands + 2 spectra), no flush" if bits >= 1 << 28
            else "working set may be L2-resident (small config)",
            "paper_ms_haswell": PAPER_MS.get(args.config),
            "timing": "headline: CUDA events around exactly `steps` multiplies, no profiling hooks; per-kernel "
                      f"breakdown (`kernels`, roofline durations): a separate run of {nprof} multiplies with a CUDA "
                      "event pair around every launch",
            **({"cuda_graph": True, "ms_per_step_eager": round(ms_eager / args.steps, 4)} if ms_eager is not None else {}),
        },
        "roofline": roof,
        "kernels": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()} for r in prof],
        "kernels_steps": nprof,
        "clocks": clocks,
        "e2e": {"value": round(e2e_val, 4), "unit": UNIT, "h2d_bytes_per_step": ha_bytes + hb_bytes,
                "d2h_bytes_per_step": hc_bytes, "ms_per_step": round(e2e_ms / args.e2e_steps, 4),
                "steps": args.e2e_steps, "per_rank_bytes": sharded,
                "pipelined": "H2D / multiply / D2H of consecutive steps overlap (2 buffer sets, separate copy streams)"},
        "gpu_launches": launches * args.steps,
    }
    if companion:
        line["companion"] = companion
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, bits, batch, args.alg)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if sharded:
        comm.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
