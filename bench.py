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

    # inputs for every step, resident in HBM before timing
    steps_total = args.warmup + args.steps
    batches = []
    for i in range(steps_total):
        start, cnt = shard(w.n_pulses, B, i, rank, world)
        o, d, t = w.pulses(start, cnt)
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        batches.append((start, to(o), to(d), to(t)))
    # device outputs of the timed steps: dense waveform rows (default), the
    # lossless packed support rows, or neither (binning still runs)
    out = h.alloc_outputs(B, hp, device=dev, waveform=args.waveform == "dense",
                          compact=args.waveform == "compact",
                          compact_capacity=B * n_bins if args.waveform == "compact" else None)
    torch.cuda.synchronize()

    def step(i, st=False, counters=False):
        start, o, d, t = batches[i]
        return h.simulate(scene, hp, o, d, t, pulse_index_base=start, outputs=out,
                          stats=st, counters=counters)[1]

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    trace_ms = wave_ms = 0.0
    launches = trace_launches = 0
    ev0.record(stream)
    for i in range(args.warmup, steps_total):
        st = step(i, st=True)
        trace_ms += st.trace_ms
        wave_ms += st.waveform_ms
        launches += st.kernel_launches
        trace_launches += st.trace_launches
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    ms_max = max_over_ranks(ms, world, dev)

    subrays = B * N * args.steps * world
    pulses = B * args.steps * world
    value = subrays / (ms_max / 1e3) / 1e6

    # ---- algorithmic bytes (instrumented, untimed re-run of the same batches)
    nodes = tris = vox = f64 = beam_nodes = n_ret = 0
    node_bytes = 64
    for i in range(args.warmup, steps_total):
        st = step(i, counters=True)
        node_bytes = st.node_bytes or 64
        nodes += st.nodes_visited
        tris += st.tris_tested
        vox += st.voxel_steps
        f64 += st.fp64_tests
        beam_nodes += st.beam_nodes
        n_ret += st.returns
    sub_rank = B * N * args.steps
    # per subray: nodes K6 tests, triangles, voxel steps; per pulse: nodes the
    # beam pre-pass K6a tests (once for all the pulse's subrays)
    b_ray = node_bytes * nodes + 48 * tris + 4 * vox + 64 * beam_nodes
    b_trace = b_ray + 24 * B * args.steps + 16 * sub_rank  # + pulse inputs + records
    b_pulse = (32 + 8 + 1 + 4 * n_bins + 32 * p.max_returns) * B * args.steps
    peak, peak_src = peaks()
    ach_trace = b_trace / (trace_ms / 1e3) / 1e9
    n_trace_launches = max(1, trace_launches)
    traffic, limiter, issue = None, None, None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f).get(args.config)
        if tj:
            kt = tj["k_trace"]
            traffic = kt["dram_bytes"] / kt["units"] * (sub_rank / n_trace_launches)
            limiter = {"issue_slots_busy": kt["issue_slots_busy"],
                       "dram_bytes_per_subray": kt["dram_bytes"] / kt["units"],
                       "l1_hit": kt["l1_hit"], "source": tj["source"]}
            if "warp_inst" in kt:
                # the bound that binds: SM instruction issue (4 warp instructions
                # per clock per SM).  Warp instructions per subray of K6a + K6 and
                # per pulse of K7 from the ncu capture, times this step's subrays
                # and pulses, over the step time (the kernels overlap on several
                # streams, so the whole step is the unit)
                wi = kt["warp_inst"] / kt["units"]
                kw = tj.get("k_waveform", {})
                wp = kw["warp_inst"] / kw["units"] if "warp_inst" in kw else 0.0
                sms = torch.cuda.get_device_properties(dev).multi_processor_count
                mhz = (clk or {}).get("sm_mhz") or 1965.0
                peak_issue = sms * 4 * mhz * 1e6
                ach = (wi * sub_rank + wp * B * args.steps) / (ms / 1e3)
                issue = {"bound": "issue", "kernel": "k_beam + k_trace + k_waveform (whole step)",
                         "achieved": ach / 1e9, "peak": peak_issue / 1e9,
                         "unit": "G warp-instructions/s", "frac": ach / peak_issue,
                         "warp_inst_per_subray": wi, "waveform_warp_inst_per_pulse": wp,
                         "source": tj["source"]}
    except Exception:
        pass
    r1 = (b_ray + b_pulse) / (ms / 1e3) / 1e9 / peak

    # ---- the same device-resident steps with the lossless packed outputs
    # (packed returns + packed waveform support rows instead of 7 fixed return
    # slots and dense rows: the zero fill of dense rows is HBM traffic, 10.7 KB
    # per pulse on C4)
    packed = None
    if args.waveform == "dense" and not args.no_packed:
        pout = h.alloc_outputs(B, hp, device=dev, waveform=False, compact=True,
                               compact_capacity=B * n_bins, packed_returns=True, slots=False,
                               returns_capacity=B * p.max_returns)
        for i in range(min(args.warmup, 2)):
            start, o, d, t = batches[i]
            h.simulate(scene, hp, o, d, t, pulse_index_base=start, outputs=pout)
        torch.cuda.synchronize()
        barrier(world)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.warmup, steps_total):
            start, o, d, t = batches[i]
            h.simulate(scene, hp, o, d, t, pulse_index_base=start, outputs=pout)
        e1.record(stream)
        torch.cuda.synchronize()
        pms = max_over_ranks(e0.elapsed_time(e1), world, dev)
        packed = {"value": subrays / (pms / 1e3) / 1e6, "unit": "Mrays/s",
                  "ms_per_step": pms / args.steps,
                  "outputs": "packed returns + packed waveform support rows (lossless)"}
        del pout

    # ---- end to end through the C ABI with host buffers (copies inside):
    # every step copies its pulses host->device and the full result back
    # (returns + the complete waveform, as lossless packed support rows; the
    # dense-row variant is reported beside it)
    e2e = e2e_dense = None
    if not args.no_e2e:
        def run_e2e(compact):
            start, o, d, t = batches[args.warmup]
            ho, hd, ht = (x.cpu().pin_memory() for x in (o, d, t))
            hout = h.alloc_outputs(B, hp, device="cpu", waveform=not compact, pin_memory=True,
                                   compact=compact,
                                   compact_capacity=B * n_bins if compact else None,
                                   packed_returns=compact, slots=not compact,
                                   returns_capacity=B * p.max_returns if compact else None)
            h.simulate(scene, hp, ho, hd, ht, pulse_index_base=start, outputs=hout)
            torch.cuda.synchronize()
            barrier(world)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.steps):
                h.simulate(scene, hp, ho, hd, ht, pulse_index_base=start, outputs=hout)
            e1.record(stream)
            torch.cuda.synchronize()
            ems = max_over_ranks(e0.elapsed_time(e1), world, dev)
            h2d = B * (12 + 12 + 8)
            d2h = B * (1 + 8)
            if compact:  # packed returns + packed waveform rows, with their offsets
                d2h += 16 * (B + 1) + 32 * int(hout.return_offset[-1]) + \
                    4 * int(hout.wf_offset[-1])
            else:
                d2h += 32 * p.max_returns * B + 4 * n_bins * B
            del hout
            return {"value": B * N * args.steps * world / (ems / 1e3) / 1e6, "unit": "Mrays/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "pulses_per_s": B * args.steps * world / (ems / 1e3),
                    "waveform_output": "packed support rows + packed returns (lossless)"
                    if compact else "dense rows + fixed return slots"}
        e2e = run_e2e(True)
        e2e_dense = run_e2e(False)

    # ---- on-device pulse generation (helios_simulate_survey, NEXT f2): the
    # same pulses, generated from the workload's flight-line description, no
    # pulse arrays at all; device-resident outputs (as `value`) and, end to
    # end, host outputs with packed waveform rows (as `e2e`)
    survey = None
    if w.surveys and not args.no_survey:
        def seg_of(start):
            for sv, g0, cnt in w.surveys:
                if g0 <= start < g0 + cnt:
                    return sv, start - g0, min(B, g0 + cnt - start)
            return None
        segs = [seg_of(batches[i][0]) for i in range(steps_total)]
        if all(sg is not None and sg[2] == B for sg in segs):
            def sstep(i, outs):
                sv, first, cnt = segs[i]
                h.simulate_survey(scene, hp, sv, first, cnt, batches[i][0], outputs=outs)
            for i in range(args.warmup):
                sstep(i, out)
            torch.cuda.synchronize()
            barrier(world)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for i in range(args.warmup, steps_total):
                sstep(i, out)
            e1.record(stream)
            torch.cuda.synchronize()
            sms = max_over_ranks(e0.elapsed_time(e1), world, dev)
            survey = {"value": B * N * args.steps * world / (sms / 1e3) / 1e6, "unit": "Mrays/s",
                      "ms_per_step": sms / args.steps,
                      "pulses": "generated on the device from the flight lines (R30)"}
            if not args.no_e2e:
                hout = h.alloc_outputs(B, hp, device="cpu", waveform=False, pin_memory=True,
                                       compact=True, compact_capacity=B * n_bins,
                                       packed_returns=True, slots=False,
                                       returns_capacity=B * p.max_returns)
                sstep(args.warmup, hout)
                torch.cuda.synchronize()
                barrier(world)
                e0.record(stream)
                for i in range(args.steps):
                    sstep(args.warmup, hout)
                e1.record(stream)
                torch.cuda.synchronize()
                ems = max_over_ranks(e0.elapsed_time(e1), world, dev)
                d2h = B * (1 + 8) + 16 * (B + 1) + 32 * int(hout.return_offset[-1]) + \
                    4 * int(hout.wf_offset[-1])
                survey["e2e"] = {"value": B * N * args.steps * world / (ems / 1e3) / 1e6,
                                 "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                                 "d2h_bytes_per_step": d2h,
                                 "waveform_output": "packed support rows + packed returns "
                                                    "(lossless)"}
                del hout

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        n_p, sec = oracle_sample(w, threads, args.cpu_budget)
        cpu = {"value": n_p * N / sec / 1e6, "unit": "Mrays/s", "cores": threads,
               "kind": "oracle",
               "sample": f"{n_p} random pulses of {args.config} ({n_p * N} subrays), "
                         f"fp64 brute-force oracle, {sec:.1f} s on {threads} threads",
               "pulses_per_s": n_p / sec}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mrays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 decisions / f32 storage",
            "data": "synthetic (seeded generators, workloads/; paper datasets unavailable)",
            "pulses_per_s": pulses / (ms_max / 1e3),
            # discrete returns of the timed steps (rank 0 counts, instrumented re-run; x world)
            "returns_per_s": n_ret * world / (ms_max / 1e3),
            "config": {"workload": args.config, "pulses_per_step_per_gpu": B,
                       "subrays_per_pulse": N, "n_tris": w.scene.n_tris,
                       "n_bins": n_bins, "l2": "inputs larger than L2 (scene + outputs)",
                       "bvh_nodes": info.n_nodes, "bvh_depth": info.max_depth,
                       "build_ms": round(info.build_ms, 2), "gen_s": round(t_gen, 1),
                       "fit_echo_width": int(args.fit_echo_width),
                       "waveform_output": args.waveform,
                       "range_noise_sd_m": args.range_noise},
            "roofline": {"bound": "hbm", "kernel": "k_beam + k_trace", "achieved": ach_trace,
                         "peak": peak, "unit": "GB/s", "frac": ach_trace / peak,
                         "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_launch": b_trace / n_trace_launches,
                         "avg_launch_ms": trace_ms / n_trace_launches,
                         "ncu_limiter": limiter,
                         "issue_roofline": issue,
                         "share_of_step": trace_ms / ms if ms > 0 else None,
                         "waveform_share_of_step": wave_ms / ms if ms > 0 else None,
                         "nodes_per_ray": nodes / sub_rank, "node_bytes": node_bytes,
                         "beam_nodes_per_pulse": beam_nodes / (B * args.steps),
                         "tris_per_ray": tris / sub_rank,
                         "voxel_steps_per_ray": vox / sub_rank,
                         "fp64_tests_per_ray": f64 / sub_rank,
                         "step_R1": r1},
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
            "e2e_dense_rows": e2e_dense,
            "packed_outputs": packed,
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
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--ref-budget", type=float, default=12.0,
                    help="seconds of oracle work per --impl reference step")
    args = ap.parse_args()
    args.config = args.config.upper()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
