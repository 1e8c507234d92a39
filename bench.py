"""Benchmark: gate-cycle evaluations per second of the windowed re-simulation
hot path on 1..8 B200 (one process per GPU), with roofline, CPU baseline,
in-bench parity gate and end-to-end numbers.  Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload: at N = 1 the C3 roofline-study config -- 1M gates x
100,000 cycle windows, the largest single-GPU config of BASELINE.json; at
N > 1 the C4 config (10M gates), weak scaling: each rank simulates a fixed
share of windows, the shards cut by ``distributed.shard_windows`` at equal
shares of per-window input activity.

A step = one pass of the hot path over the rank's windows: per window chunk
K1 stimulus segmentation + one K4 gate-eval launch per (level, fanin group)
with the toggle/dwell reduction fused, per-net sums accumulated on the device,
and (N > 1) one NCCL all-reduce of those sums (``gs_allreduce_stats``).  ``value`` has the stimulus
already resident in HBM (generated there, bit-identical to synth.stimulus);
``e2e`` takes it from pinned host memory through the C ABI every step
(gs_stim_create: H2D + device validation) and reads the sums back.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "gate-cycle evals/sec (whole box)"
UNIT = "gate-cycle evals/s"
C4_WINDOWS_PER_GPU = 16384


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="", help="C2/C3/C4/C5-... (default C3 at N=1, C4 at N>1)")
    ap.add_argument("--windows", type=int, default=0, help="windows per GPU (0 = the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="end-to-end steps (0 = as many as --steps)")
    ap.add_argument("--cpu-windows", type=int, default=0,
                    help="CPU baseline / parity sample windows (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["hbm_gbs"], "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def host_cpu():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class RcaConfig:
    """the 20-bit ripple-carry adder, 1k windows, full SDF,
    built from its text documents through the parsers (synth.rca_docs)."""
    name = "C1"
    description = ("small combinational netlist (20-bit ripple-carry adder, 100 gates), "
                   "1k cycles, full SDF (COND + INTERCONNECT), text documents")
    windows = 1000
    pct = 100
    averaged = False
    ppis = 0

    def __init__(self):
        import paper_2203_06117_b200 as api
        from paper_2203_06117_b200 import synth
        lib_t, net_t, sdf_t, vcd_t, period = synth.rca_docs()
        nl = api.parse_netlist(net_t, api.parse_library(lib_t))
        lv = api.levelize(nl)
        delays = api.parse_sdf(sdf_t, nl)
        waves, duration = api.parse_vcd(vcd_t, nl)
        b = api.window_boundaries(duration, period=period)
        self.stim = api.StimulusSet.build(waves, nl, b)
        self.model = api.compile_design(lv, delays)
        self.period = period
        self.gates = nl.num_gates
        self.levels = lv.num_levels
        self.num_inputs = nl.num_pis


def is_rca(cfg):
    return getattr(cfg, "name", "") == "C1"


def design_of(cfg):
    from paper_2203_06117_b200 import synth
    return cfg.model if is_rca(cfg) else synth.design(cfg)


def host_stimulus(cfg, lo, hi):
    """Per-input CSR stimulus of windows [lo, hi) (the oracle's input)."""
    from paper_2203_06117_b200 import synth
    if is_rca(cfg):
        assert (lo, hi) == (0, cfg.windows), "C1 runs its whole stimulus"
        return cfg.stim
    return synth.stimulus(cfg, lo, hi)


def device_stimulus(cfg, dev, lo, hi):
    from paper_2203_06117_b200 import _native
    if is_rca(cfg):
        return _native.Stimulus(dev, host_stimulus(cfg, lo, hi))
    return _native.SynthStimulus(dev, cfg, lo, hi)


def pick_config(args, world):
    from paper_2203_06117_b200 import synth
    name = args.config or ("C3" if world == 1 else "C4")
    if name == "C1":
        cfg = RcaConfig()
        return cfg, cfg.windows
    cfg = synth.config(name)
    if args.windows:
        per_gpu = args.windows
    elif name == "C4":
        per_gpu = C4_WINDOWS_PER_GPU
    else:
        per_gpu = cfg.windows
    return cfg, per_gpu


def cpu_sample_windows(args, cfg):
    """Windows of the CPU baseline / parity sample: ~1e8 gate-windows."""
    if args.cpu_windows:
        return args.cpu_windows
    return int(max(4, min(2048, 1.0e8 // cfg.gates)))


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu),
                                          f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
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
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU legs

def oracle_run(cfg, model, w_lo, w_hi, threads):
    """The reference algorithm on the host (oracle port: the reference's
    windowing, count pass, store pass and dwell_sweep restated in C/numpy,
    OpenMP) over absolute windows [w_lo, w_hi) of the config: (stats dict,
    arena dict, seconds).  Timed: StimulusSet.build's windowing of the
    per-input waveforms (WF:243-265, as the reference's Python loop), both
    passes and compute_stats -- the reference's path from per-input
    waveforms to per-net statistics."""
    from oracle import port
    port.build()
    m = model
    d = port.Design.from_arrays(m.num_pis, m.order, m.level_starts, m.pin_off, m.pin_net,
                                m.pin_ic, m.pin_arc, m.arc_rows, m.lut_off, m.lut_bits)
    s = host_stimulus(cfg, w_lo, w_hi)
    t0 = time.perf_counter()
    st = port.Stimulus.from_csr(s.pi_off, s.pi_times, s.pi_init, s.boundaries)
    arena = port.two_pass_simulate(d, st, pct=cfg.pct, threads=threads)
    stats = port.compute_stats(d, st, arena, threads=threads)
    dt = time.perf_counter() - t0
    return stats, arena, dt


def run_reference_arm(args, rank, world):
    """--impl reference: the reference algorithm (oracle port, all host
    cores) on this config's workload; rank 0 only, a bounded window sample
    per step."""
    if rank != 0:
        return
    from paper_2203_06117_b200 import synth
    cfg, per_gpu = pick_config(args, world)
    threads = os.cpu_count() or 1
    sample = min(cpu_sample_windows(args, cfg), per_gpu)
    m = design_of(cfg)
    times = []
    for i in range(args.warmup + args.steps):
        lo = (i * sample) % max(1, per_gpu - sample + 1)
        _, _, dt = oracle_run(cfg, m, lo, lo + sample, threads)
        if i >= args.warmup:
            times.append(dt)
    dt = statistics.median(times)
    v = cfg.gates * sample / dt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference",
            "config": {**config_desc(cfg, per_gpu, world), "sample_windows_per_step": sample},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu": host_cpu(),
                             "sample": f"{cfg.name} design, {sample} consecutive windows per "
                                       "step: oracle/port.py (the reference's algorithm "
                                       "restated in C + numpy, OpenMP; the reference itself is "
                                       "numba and does not travel to the GPU box) -- "
                                       "windowing, count + store pass, dwell sweep; rate "
                                       "extrapolates linearly (windows are independent)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def pinned_copy(a):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t.numpy()


def config_desc(cfg, windows_per_gpu, world):
    return {"workload": f"{cfg.name}: {cfg.description}", "gates": cfg.gates,
            "levels": cfg.levels, "inputs": cfg.num_inputs, "windows_per_gpu": windows_per_gpu,
            "windows_total": windows_per_gpu * world, "period_fs": cfg.period,
            "pathpulse_pct": cfg.pct,
            "delay_mode": "averaged" if cfg.averaged else "full conditional",
            "parallelism": f"windows sharded x{world}" if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (each step streams tens of GB of waveform/count "
                  "arrays through HBM; no flush needed)"}


# ---------------------------------------------------------------- GPU arm

def algorithmic_bytes(model, windows, input_toggles, output_toggles):
    """SURVEY §8(d) bytes of K4 over a whole step:
    sum over gate-windows of  sum_p (4 + 4 n_in(p)) + (4 + 4 n_out) + (k+1)/8."""
    sum_k = int(model.pin_off[-1])
    G = model.num_gates
    return (4 * sum_k * windows + 4 * input_toggles + 4 * G * windows + 4 * output_toggles
            + (sum_k + G) * windows / 8.0)


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    import torch.distributed as dist
    from paper_2203_06117_b200 import _native, distributed

    torch.cuda.set_device(local)
    _native.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg, per_gpu = pick_config(args, world)
    total = per_gpu * world
    weights = (_native.synth_window_counts(cfg, 0, total, local) + 1
               if world > 1 and not is_rca(cfg) else None)
    w_lo, w_hi = distributed.shard_windows(total, world, rank, weights)
    Wr = w_hi - w_lo
    model = design_of(cfg)
    N = model.num_nets

    stream = torch.cuda.Stream()
    dev = model.device()
    dstim = device_stimulus(cfg, dev, w_lo, w_hi)   # resident in HBM
    eng = _native.Engine(dev, 0, stream.cuda_stream)
    acc = torch.zeros(3 * N + 3, dtype=torch.int64, device="cuda")

    comm = distributed.nccl_comm(device=local) if world > 1 else None

    def step(s):
        acc.zero_()
        eng.run_stats_device(s, 0, Wr, cfg.pct, acc.data_ptr())
        if world > 1:  # the library's NCCL all-reduce of the device sums
            comm.allreduce_stats(acc.data_ptr(), acc.numel(), stream.cuda_stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(dstim)
        torch.cuda.synchronize()
        sampler = ClockSampler(local)
        sampler.start()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eval_ms = 0.0
        launches = 0
        for _ in range(args.steps):
            step(dstim)
            t = eng.timing()
            eval_ms += t["ms_gate_eval"]
            launches += t["launches"] + t["chunks"]
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = sampler.stop()
        ms = e0.elapsed_time(e1)
        timing = eng.timing()
        acc_value = acc.clone()

        # ---- end to end through the C ABI with host buffers: pinned host CSR
        # stimulus -> device (gs_stim_create), run, per-net sums -> host
        from paper_2203_06117_b200.waveform import StimulusSet
        if is_rca(cfg):
            hs = host_stimulus(cfg, w_lo, w_hi)
            hb, hoff, htimes, hinit = (pinned_copy(a) for a in
                                       (hs.boundaries, hs.pi_off, hs.pi_times, hs.pi_init))
        else:
            hb, hoff, htimes, hinit = dstim.download(pinned=True)
        hstim = StimulusSet.from_csr(hb, hoff, htimes, hinit)
        h2d = hb.nbytes + hoff.nbytes + htimes.nbytes + hinit.nbytes
        d2h = acc.numel() * 8
        host_acc = torch.empty(acc.numel(), dtype=torch.int64).pin_memory()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        # serial breakdown of one step (second of two: the stimulus pool is
        # warm): upload, then simulate and read back
        for _ in range(2):
            h0 = time.perf_counter()
            s2 = _native.Stimulus(dev, hstim)          # H2D of this step's stimulus
            h1 = time.perf_counter()
            step(s2)
            host_acc.copy_(acc, non_blocking=True)     # D2H of the per-net sums
            stream.synchronize()
            h2 = time.perf_counter()
            del s2
        e2e_upload_ms, e2e_run_ms = 1e3 * (h1 - h0), 1e3 * (h2 - h1)
        # end to end, as a streaming user runs it: step i+1's stimulus upload
        # (gs_stim_create: pinned H2D + device validation, on its own stream
        # from a worker thread) overlaps step i's simulation; every step still
        # uploads its inputs and reads its sums back inside the timed region
        from concurrent.futures import ThreadPoolExecutor
        K = max(1, args.e2e_steps or args.steps)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ThreadPoolExecutor(1) as ex:
            fut = ex.submit(_native.Stimulus, dev, hstim)
            s_w = _native.Stimulus(dev, hstim)
            step(s_w)
            stream.synchronize()
            del s_w
            fut.result()
            del fut
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fut = ex.submit(_native.Stimulus, dev, hstim)
            for i in range(K):
                s_i = fut.result()
                if i + 1 < K:
                    fut = ex.submit(_native.Stimulus, dev, hstim)
                step(s_i)
                host_acc.copy_(acc, non_blocking=True)
                stream.synchronize()
                del s_i
            t1 = time.perf_counter()
        e2e_ms = 1e3 * (t1 - t0) / K
        e2e_same = bool(torch.equal(host_acc, acc_value.cpu()))
        del hstim, hb, hoff, htimes, hinit

    # max over ranks
    tm = torch.tensor([ms, e2e_ms, eval_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms, e2e_ms, eval_ms = tm.tolist()
    ms_step = ms / args.steps
    units = cfg.gates * total
    value = units / (ms_step / 1e3)
    e2e_value = units / (e2e_ms / 1e3)

    # roofline of K4 on this rank's windows (identical every step).  Toggle
    # totals from this rank's per-net counts: n_in = sum over pins of the
    # driving net's toggles, n_out = gate-net toggles.
    acc.zero_()
    eng.run_stats_device(dstim, 0, Wr, cfg.pct, acc.data_ptr())
    tc_net = acc[N:2 * N].cpu().numpy()
    fanout = np.bincount(model.pin_net, minlength=N)
    in_tog = int((tc_net * fanout).sum())
    out_tog = int(tc_net[model.num_pis:].sum())
    hbm, peak_src = peaks()
    bytes_step = algorithmic_bytes(model, Wr, in_tog, out_tog)
    k4_ms = eval_ms / args.steps
    achieved = bytes_step / (k4_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k4_traffic.json")
    if os.path.exists(prof):
        try:
            for ent in json.load(open(prof)):
                if ent.get("config") == cfg.name and ent.get("windows") == Wr:
                    traffic = ent.get("dram_bytes_per_launch")
        except Exception:
            pass

    # parity gate and CPU baseline (rank 0, N = 1): the oracle on a sample of
    # this run's windows against the device's per-net sums for the same
    # windows
    cpu = parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        S = min(cpu_sample_windows(args, cfg), Wr)
        ref, arena, dt = oracle_run(cfg, model, w_lo, w_lo + S, threads)
        got = eng.run_stats(dstim, 0, S, cfg.pct)
        tot = (int(arena["filtered"].sum()), int(arena["ic_filtered"].sum()),
               int(arena["discarded"].sum()))
        t0g = (int(ref["duration"]) - got[0])
        ok = (np.array_equal(got[0], ref["t1"]) and np.array_equal(t0g, ref["t0"])
              and np.array_equal(got[1], ref["tc"]) and np.array_equal(got[2], ref["ig"])
              and tuple(got[3]) == tot)
        parity = {"result": "ok" if ok else "MISMATCH", "windows": [w_lo, w_lo + S],
                  "nets": N, "checked": "per-net T0/T1/TC/IG and filtered/ic_filtered/"
                  "discarded totals, device run vs oracle/port.py, bit-exact",
                  "e2e_sums_equal_value_sums": e2e_same}
        r = cfg.gates * S / dt
        cpu = {"value": r, "unit": UNIT, "cores": threads, "kind": "port", "cpu": host_cpu(),
               "sample": f"{cfg.name} design, windows [{w_lo},{w_lo + S}) ({S} of {Wr}; "
                         f"linear extrapolation, windows are independent): oracle/port.py, "
                         f"the reference algorithm restated in C + numpy with OpenMP (the "
                         f"numba reference does not travel to the GPU box) -- windowing, "
                         f"count + store pass, dwell sweep -- on {threads} host threads, "
                         f"{dt:.1f} s"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "int64", "data": "synthetic (counter-based RNG stimulus generated "
                                          "on the device, random-init design of the "
                                          "config's shape)",
                "config": config_desc(cfg, per_gpu, world),
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                             "frac": achieved / hbm, "traffic": traffic,
                             "kernel": "gate_eval (K4)", "peak_source": peak_src,
                             "algorithmic_bytes_per_step": bytes_step,
                             "k4_ms_per_step": k4_ms,
                             "k4_launches_per_step": timing["gate_eval_launches"],
                             "bytes_per_gate_window": bytes_step / (cfg.gates * Wr)},
                "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                        "steps": K, "stat": "wall clock over the steps / steps (step i+1's "
                        "upload overlapped with step i)", "serial_ms_per_step":
                        e2e_upload_ms + e2e_run_ms,
                        "host_ms_stim_upload": e2e_upload_ms, "host_ms_run": e2e_run_ms},
                "clocks": clocks, "gpu_launches": launches,
                "cuda_graphs": {"chunk_graphs_built": timing["graph_builds"],
                                "chunk_graph_replays": timing["graph_replays"],
                                "note": "each window chunk's launch sequence (K1 + every "
                                        "level's K4 launches) is one CUDA graph, built on "
                                        "first use and replayed"},
                "activity": {"input_toggles_per_gw": in_tog / (cfg.gates * Wr),
                             "output_toggles_per_gw": out_tog / (cfg.gates * Wr),
                             "chunks_per_step": timing["chunks"]}}
        if world > 1:
            line["shards"] = "distributed.shard_windows over per-window input activity"
        if parity is not None:
            line["parity"] = parity
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
        if parity is not None and parity["result"] != "ok":
            sys.exit(3)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
