"""bench.py -- throughput of the HELIOS++ hot path on B200 (BASELINE.json metric:
"Mrays/s traced and pulses/s with full waveform on 1 B200; % of HBM roofline").

One step = one batch of pulses of the workload through the whole hot path
(subray fan-out, LBVH/voxel trace, radiometry, full waveform, peaks) via
helios_simulate.  Inputs are resident in HBM when the timed region starts.
Multi-GPU: one process per GPU (torchrun), each rank simulates its own pulse
ranges of the same scene (pulses are independent: no collective on the data
path, "scaling": "weak"); time = max over ranks of CUDA-event time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--batch B]
  python bench.py --impl reference ...   # the fp64 CPU oracle on host cores

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mrays/s traced and pulses/s with full waveform on 1 B200; % of HBM roofline"
DEFAULT_BATCH = {"C1": 10_000, "C2": 1_000_000, "C3": 1_000_000, "C4": 1_000_000,
                 "C5": 1_000_000, "C6": 1_000_000}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows)}


def dist_setup(backend):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
    return rank, world, local


def shard(n_pulses: int, batch: int, step: int, rank: int, world: int):
    """Pulse range of (step, rank): disjoint contiguous batches, rank-major
    within a step, wrapping around the workload."""
    nb = max(1, n_pulses // batch)
    g = (step * world + rank) % nb
    return g * batch, min(batch, n_pulses - g * batch)


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------ CPU oracle
def oracle_sample(w, n_threads: int, budget_s: float, seed: int = 0):
    """Time the oracle (as it stands) on a bounded random sample of the
    workload's pulses, sized to ~budget_s of wall time on n_threads host
    threads (calibrated on a small first sample); returns (pulses, seconds)."""
    import oracle
    rng = np.random.default_rng(seed)
    k = 1
    while True:
        ids = np.sort(rng.choice(w.n_pulses, k, replace=False))
        o, d, t = w.pulses_at(ids)
        t0 = time.perf_counter()
        oracle.simulate(w.scene, w.params, o, d, t, ids.astype(np.uint64), n_threads=n_threads)
        dt = time.perf_counter() - t0
        if dt >= 0.4 * budget_s or k >= 2_000_000:
            return k, dt
        k = int(min(2_000_000, max(2 * k, k * 0.8 * budget_s / max(dt, 1e-3))))


def run_reference(args):
    rank, world, _ = dist_setup("gloo")
    if rank != 0:
        return 0
    from workloads import make_workload
    import oracle
    oracle.build()
    w = make_workload(args.config)
    N = w.params.subray_count
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(1)
    # each step: a bounded random sample of the workload, sized so that the
    # whole --warmup + --steps run takes about 2.5 minutes of oracle work
    budget = max(1.0, min(args.ref_budget, 150.0 / max(1, args.steps + args.warmup)))
    per_step, _ = oracle_sample(w, threads, budget, seed=123)
    times = []
    for i in range(args.warmup + args.steps):
        ids = np.sort(rng.choice(w.n_pulses, per_step, replace=False))
        o, d, t = w.pulses_at(ids)
        t0 = time.perf_counter()
        oracle.simulate(w.scene, w.params, o, d, t, ids.astype(np.uint64), n_threads=threads)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    T = sum(times)
    value = per_step * N * args.steps / T / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mrays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * T / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generators, workloads/)",
        "pulses_per_s": per_step * args.steps / T,
        "config": {"workload": args.config, "pulses_per_step": per_step, "subrays": N,
                   "n_tris": w.scene.n_tris},
        "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads, "kind": "oracle",
                         "sample": f"{per_step} random pulses of {args.config} per step, "
                                   f"brute-force fp64 oracle, {threads} threads"},
        "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
DENSE_OUT_BUDGET = 96e9   # device bytes of dense output sets one multi-batch call may use
PACKED_FLOATS_PER_PULSE = 192  # packed waveform capacity per pulse (grown on demand)


def _groups(idx, m):
    return [idx[i:i + m] for i in range(0, len(idx), m)]


def run_ours(args):
    import torch
    rank, world, local = dist_setup("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2101_09154_b200 as h
    from paper_2101_09154_b200 import build as hb
    if not hb.up_to_date():
        if rank == 0:
            hb.build()
        barrier(world)
    from workloads import make_workload

    t_gen = time.perf_counter()
    w = make_workload(args.config)
    t_gen = time.perf_counter() - t_gen
    from dataclasses import replace as _replace
    w.params = _replace(w.params, fit_echo_width=int(args.fit_echo_width),
                        range_noise_sd_m=args.range_noise)
    p = w.params
    N = p.subray_count
    hp = h.make_params(p)
    n_bins = h.helios_waveform_bins(hp)
    B = min(args.batch or DEFAULT_BATCH[args.config], w.n_pulses)
    scene = h.Scene.from_workload_scene(w.scene, device=dev)
    info = scene.info()
    stream = torch.cuda.current_stream()
    fp64_tflops = h.util_fp64_fma_tflops()

    # inputs for every step (distinct batches), resident in HBM before timing
    steps_total = args.warmup + args.steps
    batches = []
    for i in range(steps_total):
        start, cnt = shard(w.n_pulses, B, i, rank, world)
        o, d, t = w.pulses(start, cnt)
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        batches.append((to(o), to(d), to(t), start))
    dense = args.waveform == "dense"
    out_bytes = B * (4 * n_bins * dense + 32 * p.max_returns + 9)
    # output sets the timed steps rotate through (one per batch of a call):
    # --out-sets (default 2: a batch's outputs are overwritten two steps later,
    # D-4 "outputs are overwritten per batch"), capped by the device budget
    M = max(1, min(args.steps, args.out_sets, int(DENSE_OUT_BUDGET // max(1, out_bytes))))
    outs = [h.alloc_outputs(B, hp, device=dev, waveform=dense,
                            compact=args.waveform == "compact",
                            compact_capacity=B * n_bins if args.waveform == "compact" else None)
            for _ in range(M)]
    torch.cuda.synchronize()

    def run_steps(idx, st=False, counters=False):
        """The steps idx through helios_simulate_batches, <= M batches per call
        (each with its own output set); stats summed."""
        tot = {}
        for g in _groups(list(idx), M):
            r = h.simulate_batches(scene, hp, [batches[i] for i in g], outs[:len(g)],
                                   stats=st, counters=counters)
            if r is not None:
                for f, _ in r._fields_:
                    tot[f] = tot.get(f, 0) + getattr(r, f)
        return tot

    def timed(fn):
        barrier(world)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(e0.elapsed_time(e1), world, dev), r

    # non-blocking calls (helios_simulate_batches_async): one batch per call,
    # two calls in flight on two streams, each with its own output set, so a
    # call's tail (its last K7) overlaps the next call's head (K6a, K6).  The
    # streams wait for the timing event first; every call is waited for before
    # the end event is recorded.
    astreams = [torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)]

    def run_steps_async(idx, st=False):
        tot = {}
        pending = []
        for s_ in astreams:
            s_.wait_stream(stream)
        for j, i in enumerate(idx):
            if len(pending) == 2:
                r = pending.pop(0).wait()
                if r is not None:
                    for f, _ in r._fields_:
                        tot[f] = tot.get(f, 0) + getattr(r, f)
            pending.append(h.simulate_batches_async(scene, hp, [batches[i]], [outs[j % M]],
                                                    stream=astreams[j % 2], stats=st))
        for c in pending:
            r = c.wait()
            if r is not None:
                for f, _ in r._fields_:
                    tot[f] = tot.get(f, 0) + getattr(r, f)
        return tot

    run_steps(range(args.warmup))
    torch.cuda.synchronize()
    timed_idx = range(args.warmup, steps_total)

    # ---- the timed steps: K batches of B pulses through helios_simulate_batches
    # (one chunk pipeline per call, so a batch's head overlaps the previous tail)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    use_async = args.value_api == "async" and M >= 2
    if use_async:
        run_steps_async(range(args.warmup))  # warm the two streams' scratch
        torch.cuda.synchronize()
        ms_max, st_main = timed(lambda: run_steps_async(timed_idx, st=True))
    else:
        ms_max, st_main = timed(lambda: run_steps(timed_idx, st=True))
    clk = clocks.stop()
    launches = int(st_main.get("kernel_launches", 0))
    subrays = B * N * args.steps * world
    pulses = B * args.steps * world
    value = subrays / (ms_max / 1e3) / 1e6

    # ---- the same steps as one blocking helios_simulate call each
    def blocking():
        for i in timed_idx:
            o, d, t, start = batches[i]
            h.simulate(scene, hp, o, d, t, pulse_index_base=start, outputs=outs[0])
    bms, _ = timed(blocking)

    # ---- exclusive kernel times: every kernel of the same steps on one stream
    # (helios_tuning.serialize), CUDA events around each launch (helios_stats)
    with h.tuning(serialize=1):
        sms_ser, st_ser = timed(lambda: run_steps(timed_idx, st=True))
    # ---- algorithmic bytes: instrumented kernel variant, untimed
    st_cnt = run_steps(timed_idx, counters=True)
    nodes, tris = st_cnt["nodes_visited"], st_cnt["tris_tested"]
    vox, f64, beam_nodes = st_cnt["voxel_steps"], st_cnt["fp64_tests"], st_cnt["beam_nodes"]
    n_ret = st_cnt["returns"]
    sub_rank = B * N * args.steps
    pul_rank = B * args.steps
    # B_ray = 64 N_node + 48 N_tri + 4 N_cell (+ 64 per K6a node
    # test, once per pulse for all its subrays); B_pulse = 32 + 8 + 1 + 4 n_bins + 32 R
    b_ray = 64 * nodes + 48 * tris + 4 * vox + 64 * beam_nodes
    b_pulse = (32 + 8 + 1 + 4 * n_bins + 32 * p.max_returns) * pul_rank
    # K6 (k_trace) alone: its traversal reads + pulse inputs + the 12-B records it writes
    b_k6 = 64 * nodes + 48 * tris + 4 * vox + 24 * pul_rank + 12 * sub_rank
    # K7 (k_waveform) alone: 8-B records read + row, returns, k0, count written
    b_k7 = 8 * sub_rank + (4 * n_bins * dense + 32 * p.max_returns + 9) * pul_rank
    peak, peak_src = peaks()
    k6_ms, k6a_ms, k7_ms = st_ser["trace_ms"], st_ser["beam_ms"], st_ser["waveform_ms"]
    n_launch = max(1, int(st_ser["trace_launches"]))
    ach_k6 = b_k6 / (k6_ms / 1e3) / 1e9
    ach_k7 = b_k7 / (k7_ms / 1e3) / 1e9
    r1 = (b_ray + b_pulse) / (ms_max / 1e3) / 1e9 / peak
    traffic, issue, alu = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f).get(args.config)
        if tj:
            kt = tj["k_trace"]
            traffic = kt["dram_bytes"] / kt["units"] * (sub_rank / n_launch)
            kw = tj.get("k_waveform", {})
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            mhz = (clk or {}).get("sm_mhz") or 1965.0
            peak_issue = sms * 4 * mhz * 1e6
            wi = kt["warp_inst"] / kt["units"]
            wp = kw["warp_inst"] / kw["units"] if "warp_inst" in kw else 0.0
            issue = {"bound": "issue", "achieved": (wi * sub_rank + wp * pul_rank) / (ms_max / 1e3) / 1e9,
                     "peak": peak_issue / 1e9, "unit": "G warp-instructions/s",
                     "frac": (wi * sub_rank + wp * pul_rank) / (ms_max / 1e3) / peak_issue,
                     "warp_inst_per_subray_k6a_k6": wi, "warp_inst_per_pulse_k7": wp,
                     "k6_issue_slots_busy": kt.get("issue_slots_busy"),
                     "k7_issue_slots_busy": kw.get("issue_slots_busy"),
                     "source": tj["source"]}
            if "fp64_pipe_busy" in kt:
                # K6's fp64 pipe against the FMA rate measured live by the library's
                # own microbenchmark (util_fp64_fma_tflops): the share of that peak
                # K6 uses while it runs, from the ncu capture's pipe-active fraction.
                # Every decision of the path is fp64, so this is the ALU
                # bound that matters on C4, whose DDA is fp64 throughout.
                alu = {"bound": "alu", "pipe": "fp64", "kernel": "k_trace (K6)",
                       "peak": fp64_tflops, "unit": "TFLOP/s (fp64 FMA, measured)",
                       "frac": kt["fp64_pipe_busy"],
                       "achieved": kt["fp64_pipe_busy"] * fp64_tflops if fp64_tflops else None,
                       "k6_pipe_busy": {"fp64": kt["fp64_pipe_busy"], "alu": kt.get("alu_pipe_busy"),
                                        "fma": kt.get("fma_pipe_busy")},
                       "k7_pipe_busy": {"fp64": kw.get("fp64_pipe_busy"), "alu": kw.get("alu_pipe_busy"),
                                        "fma": kw.get("fma_pipe_busy")},
                       "source": "sm__inst_executed_pipe_*.avg.pct_of_peak_sustained_active, " + tj["source"]}
    except Exception:
        pass

    # ---- the same steps with the lossless packed outputs (packed returns +
    # packed waveform support rows) instead of fixed slots and dense rows
    packed = None
    if not args.no_packed:
        pouts = [h.alloc_outputs(B, hp, device=dev, waveform=False, compact=True,
                                 compact_capacity=B * PACKED_FLOATS_PER_PULSE,
                                 packed_returns=True, slots=False,
                                 returns_capacity=B * p.max_returns) for _ in range(min(M, 8))]
        def run_packed():
            for g in _groups(list(timed_idx), len(pouts)):
                h.simulate_batches(scene, hp, [batches[i] for i in g], pouts[:len(g)])
        run_packed()  # grows capacities if needed (retry inside simulate is per call)
        pms, _ = timed(run_packed)
        packed = {"value": subrays / (pms / 1e3) / 1e6, "unit": "Mrays/s",
                  "ms_per_step": pms / args.steps,
                  "outputs": "packed returns + packed waveform support rows (lossless)"}
        del pouts

    # ---- end to end through the public API with HOST buffers: every step's
    # pulses are copied host -> device and its complete result (returns +
    # packed waveform support rows, lossless) device -> host inside the timed
    # region; distinct batches, <= 8 per helios_simulate_batches call
    e2e = None
    if not args.no_e2e:
        hb_in = []
        for i in timed_idx:
            o, d, t, start = batches[i]
            hb_in.append((o.cpu().pin_memory(), d.cpu().pin_memory(), t.cpu().pin_memory(), start))
        G = min(args.steps, 8)
        houts = [h.alloc_outputs(B, hp, device="cpu", waveform=False, pin_memory=True,
                                 compact=True, compact_capacity=B * PACKED_FLOATS_PER_PULSE,
                                 packed_returns=True, slots=False,
                                 returns_capacity=B * p.max_returns) for _ in range(G)]
        d2h = [0]

        def run_e2e():
            d2h[0] = 0
            for g in _groups(list(range(len(hb_in))), G):
                h.simulate_batches(scene, hp, [hb_in[i] for i in g], houts[:len(g)])
                for k in range(len(g)):
                    hout = houts[k]
                    d2h[0] += B * (1 + 8) + 16 * (B + 1) + 32 * int(hout.return_offset[-1]) + \
                        4 * int(hout.wf_offset[-1])
        # untimed warm-up over every host batch and output set: the first DMA
        # to / from a freshly pinned buffer costs a one-time mapping (C3: 11.8
        # vs 5.5 ms per step, tools/e2e_repro.py), and packed capacities grow
        run_e2e()
        ems, _ = timed(run_e2e)
        e2e = {"value": subrays / (ems / 1e3) / 1e6, "unit": "Mrays/s",
               "h2d_bytes_per_step": B * (12 + 12 + 8), "d2h_bytes_per_step": d2h[0] // args.steps,
               "pulses_per_s": pulses / (ems / 1e3), "ms_per_step": ems / args.steps,
               "api": f"helios_simulate_batches, {G} distinct host batches per call",
               "waveform_output": "packed support rows + packed returns (lossless)"}
        del houts, hb_in

    # ---- on-device pulse generation (helios_simulate_survey, NEXT f2): the
    # same steps generated from the workload's flight lines (no pulse arrays),
    # device-resident outputs, one blocking call per step
    survey = None
    if w.surveys and not args.no_survey:
        def seg_of(start):
            for sv, g0, cnt in w.surveys:
                if g0 <= start < g0 + cnt:
                    return sv, start - g0, min(B, g0 + cnt - start)
            return None
        segs = {i: seg_of(batches[i][3]) for i in range(steps_total)}
        if all(sg is not None and sg[2] == B for sg in segs.values()):
            def run_survey():
                for i in timed_idx:
                    sv, first, cnt = segs[i]
                    h.simulate_survey(scene, hp, sv, first, cnt, batches[i][3], outputs=outs[0])
            run_survey()
            sms, _ = timed(run_survey)
            survey = {"value": subrays / (sms / 1e3) / 1e6, "unit": "Mrays/s",
                      "ms_per_step": sms / args.steps,
                      "pulses": "generated on the device from the flight lines (R30)",
                      "api": "one blocking helios_simulate_survey per step"}

    # ---- the WHOLE configuration (every pulse of it), in
    # batches of B pulses through helios_simulate_batches (10 per call, packed
    # device outputs), 1 warm-up + 5 timed runs: median and minimum
    full = None
    if args.full_config and world == 1:
        del outs
        torch.cuda.synchronize()
        n_all = w.n_pulses
        fb = []
        for s0 in range(0, n_all, 10 * B):
            cnt = min(10 * B, n_all - s0)
            o, d, t = w.pulses(s0, cnt)
            for k in range(0, cnt, B):
                m = min(B, cnt - k)
                to = lambda a: torch.from_numpy(np.ascontiguousarray(a[k:k + m])).to(dev)
                fb.append((to(o), to(d), to(t), s0 + k))
        del batches
        G = 10
        fouts = [h.alloc_outputs(B, hp, device=dev, waveform=False, compact=True,
                                 compact_capacity=B * PACKED_FLOATS_PER_PULSE,
                                 packed_returns=True, slots=False,
                                 returns_capacity=B * p.max_returns) for _ in range(G)]

        def run_full():
            for g in _groups(list(range(len(fb))), G):
                h.simulate_batches(scene, hp, [fb[i] for i in g], [fouts[k] for k in range(len(g))])
        run_full()
        runs = [timed(run_full)[0] / 1e3 for _ in range(5)]
        full = {"pulses": n_all, "subrays": n_all * N, "batch_pulses": B, "batches_per_call": G,
                "runs_s": [round(x, 4) for x in runs], "median_s": float(np.median(runs)),
                "min_s": float(np.min(runs)),
                "Mrays_per_s_median": n_all * N / float(np.median(runs)) / 1e6,
                "pulses_per_s_median": n_all / float(np.median(runs)),
                "outputs": "packed returns + packed waveform support rows, device-resident"}
        del fouts, fb


    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n_p, sec = oracle_sample(w, threads, args.cpu_budget)
        # D-5: one thread on a small slice, extrapolated to the whole config
        n1, sec1 = oracle_sample(w, 1, max(2.0, args.cpu_budget / 4), seed=7)
        cpu = {"value": n_p * N / sec / 1e6, "unit": "Mrays/s", "cores": threads,
               "kind": "oracle",
               "sample": f"{n_p} random pulses of {args.config} ({n_p * N} subrays), "
                         f"fp64 brute-force oracle, {sec:.1f} s on {threads} threads",
               "pulses_per_s": n_p / sec,
               "one_thread": {"pulses": n1, "s": round(sec1, 2),
                              "extrapolated_full_config_s": w.n_pulses * sec1 / n1,
                              "extrapolated_full_config_s_all_cores": w.n_pulses * sec / n_p}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 decisions / f32 storage",
            "data": "synthetic (seeded generators, workloads/; paper datasets unavailable)",
            "pulses_per_s": pulses / (ms_max / 1e3),
            "returns_per_s": n_ret * world / (ms_max / 1e3),
            "config": {"workload": args.config, "pulses_per_step_per_gpu": B,
                       "subrays_per_pulse": N, "n_tris": w.scene.n_tris,
                       "n_bins": n_bins, "l2": "inputs larger than L2 (scene + outputs)",
                       "api": ("helios_simulate_batches_async, one batch (step) per call, two "
                               "calls in flight on two streams, distinct batches and output sets"
                               if use_async else
                               f"helios_simulate_batches, {M} batches (steps) per call, "
                               "distinct batches and output sets"),
                       "bvh_nodes": info.n_nodes, "bvh_depth": info.max_depth,
                       "build_ms": round(info.build_ms, 2), "gen_s": round(t_gen, 1),
                       "fit_echo_width": int(args.fit_echo_width),
                       "waveform_output": args.waveform,
                       "range_noise_sd_m": args.range_noise},
            "roofline": {"bound": "hbm", "kernel": "k_trace (K6)", "achieved": ach_k6,
                         "peak": peak, "unit": "GB/s", "frac": ach_k6 / peak,
                         "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_launch": b_k6 / n_launch,
                         "avg_launch_ms": k6_ms / n_launch,
                         "timing": "exclusive: every kernel on one stream (helios_tuning.serialize)",
                         "step_R1": r1,
                         "kernels_exclusive_ms_per_step": {
                             "k_beam (K6a)": k6a_ms / args.steps, "k_trace (K6)": k6_ms / args.steps,
                             "k_waveform (K7)": k7_ms / args.steps,
                             "serialized_step": sms_ser / args.steps},
                         "k_waveform": {"bound": "hbm", "achieved": ach_k7, "frac": ach_k7 / peak,
                                        "bytes_per_pulse": b_k7 / pul_rank},
                         "issue_roofline": issue,
                         "alu_roofline": alu,
                         "fp64_fma_tflops_measured": fp64_tflops,
                         "nodes_per_ray": nodes / sub_rank,
                         "beam_nodes_per_pulse": beam_nodes / pul_rank,
                         "tris_per_ray": tris / sub_rank,
                         "voxel_steps_per_ray": vox / sub_rank,
                         "fp64_tests_per_ray": f64 / sub_rank},
            "gpu_launches": launches,
            "clocks": clk,
            "blocking_calls": {"value": subrays / (bms / 1e3) / 1e6, "unit": "Mrays/s",
                               "ms_per_step": bms / args.steps,
                               "api": "one blocking helios_simulate per step"},
            "e2e": e2e,
            "packed_outputs": packed,
            "full_config": full,
            "device_pulse_generation": survey,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    scene.destroy()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=os.environ.get("HELIOS_BENCH_CONFIG", "C5"))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--waveform", default="dense", choices=["dense", "compact", "none"],
                    help="waveform output of the device-resident steps")
    ap.add_argument("--value-api", default="batches", choices=["batches", "async"],
                    help="timed steps through helios_simulate_batches (<= out-sets batches per "
                         "call) or helios_simulate_batches_async (one batch per call, two in "
                         "flight)")
    ap.add_argument("--out-sets", type=int, default=2,
                    help="device output sets the timed steps rotate through (batches per call)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-packed", action="store_true",
                    help="skip the device-resident packed-output measurement")
    ap.add_argument("--no-survey", action="store_true",
                    help="skip the on-device pulse generation measurement")
    ap.add_argument("--fit-echo-width", action="store_true",
                    help="optional Gaussian echo-width fit per return (P:280)")
    ap.add_argument("--range-noise", type=float, default=0.0,
                    help="ranging error sigma in m (P:288)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--full-config", type=int, default=-1,
                    help="SURVEY D-4 run over every pulse of the config (default: on for C5)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=12.0,
                    help="seconds of oracle work per --impl reference step")
    args = ap.parse_args()
    args.config = args.config.upper()
    if args.full_config < 0:
        args.full_config = 1 if args.config == "C5" else 0
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
