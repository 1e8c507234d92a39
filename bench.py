"""Benchmark: gate-cycle evaluations per second of the windowed re-simulation hot
path on 1..8 B200 (one process per GPU), with roofline, CPU baseline and
end-to-end numbers.  Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step = one pass of the hot path over this rank's window shard of the config:
K1 stimulus segmentation + one K4 gate-eval launch per logic level with the
toggle/dwell reduction fused, the per-net sums accumulated on the device, and
(N > 1) one NCCL all-reduce of those sums.  Work per GPU is fixed (weak
scaling): rank r simulates windows [r*Wc, (r+1)*Wc) of the config's stimulus.
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


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--windows", type=int, default=0, help="windows per GPU (0 = config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-windows", type=int, default=0,
                    help="CPU baseline sample windows (0 = auto)")
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

def cpu_oracle_rate(cfg, design_arrays, windows, threads, chunk=256):
    """The oracle port (reference algorithm in C + numpy, OpenMP) over windows
    [0, windows) of the config, in window chunks (exact: windows are
    independent) to bound host memory: (gate-cycle evals/s, seconds).  Timed:
    the simulation and the stats reduction (inputs prepared beforehand, like
    the GPU `value` leg)."""
    from oracle import port
    from paper_2203_06117_b200 import synth
    port.build()
    m = design_arrays
    d = port.Design.from_arrays(m.num_pis, m.order, m.level_starts, m.pin_off, m.pin_net,
                                m.pin_ic, m.pin_arc, m.arc_rows, m.lut_off, m.lut_bits)
    dt = 0.0
    for a in range(0, windows, chunk):
        b = min(windows, a + chunk)
        s = synth.stimulus(cfg, a, b)
        st = port.Stimulus.from_csr(s.pi_off, s.pi_times, s.pi_init, s.boundaries)
        t0 = time.perf_counter()
        arena = port.two_pass_simulate(d, st, pct=cfg.pct, threads=threads)
        port.compute_stats(d, st, arena, threads=threads)
        dt += time.perf_counter() - t0
        del arena, st
    return cfg.gates * windows / dt, dt


def run_reference_arm(args, cfg, rank, world):
    """--impl reference: the reference algorithm (oracle port, all host cores)
    on this config; rank 0 only."""
    if rank != 0:
        return
    from paper_2203_06117_b200 import synth
    threads = os.cpu_count() or 1
    sample = args.cpu_windows or 128
    m = synth.design(cfg)
    rates = []
    for i in range(args.warmup + args.steps):
        r, dt = cpu_oracle_rate(cfg, m, sample, threads)
        if i >= args.warmup:
            rates.append((r, dt))
    v = statistics.median(r for r, _ in rates)
    ms = statistics.median(dt for _, dt in rates) * 1e3
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "impl": "reference",
            "config": config_desc(cfg, sample),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{cfg.name} design, windows [0,{sample}) per step: "
                                       "count pass + store pass + dwell (oracle/port.py)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_desc(cfg, windows_per_gpu):
    return {"workload": f"{cfg.name}: {cfg.description}", "gates": cfg.gates,
            "levels": cfg.levels, "inputs": cfg.num_inputs, "windows_per_gpu": windows_per_gpu,
            "period_fs": cfg.period, "pathpulse_pct": cfg.pct, "delay_mode":
            "averaged" if cfg.averaged else "full conditional",
            "l2": "inputs larger than L2 (each step streams GBs of waveform/count arrays "
                  "through HBM; no flush needed)"}


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
    from paper_2203_06117_b200 import synth
    cfg = synth.config(args.config)
    if args.impl == "reference":
        return run_reference_arm(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2203_06117_b200 import _native, simcore

    torch.cuda.set_device(local)
    _native.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    Wr = args.windows or cfg.windows
    w_lo, w_hi = rank * Wr, (rank + 1) * Wr
    model = synth.design(cfg)
    stim = synth.stimulus(cfg, w_lo, w_hi)
    N = model.num_nets

    stream = torch.cuda.Stream()
    dev = model.device()
    dstim = _native.Stimulus(dev, stim)
    eng = _native.Engine(dev, 0, stream.cuda_stream)
    acc = torch.zeros(3 * N + 3, dtype=torch.int64, device="cuda")

    def step(s):
        acc.zero_()
        eng.run_stats_device(s, 0, Wr, cfg.pct, acc.data_ptr())
        if world > 1:
            dist.all_reduce(acc)

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

        # ---- end to end through the C ABI with host buffers: pinned host CSR
        # stimulus -> device (gs_stim_create), run, per-net sums -> host
        pin = {k: torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
               for k, v in (("off", stim.pi_off), ("t", stim.pi_times), ("i", stim.pi_init),
                            ("b", stim.boundaries))}
        from paper_2203_06117_b200.waveform import StimulusSet
        hstim = StimulusSet.from_csr(pin["b"].numpy(), pin["off"].numpy(), pin["t"].numpy(),
                                     pin["i"].numpy())
        h2d = sum(int(v.numel() * v.element_size()) for v in pin.values())
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
        K = max(1, args.e2e_steps)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ThreadPoolExecutor(1) as ex:
            # untimed: one overlapped step, so the stimulus pool holds two
            # stimuli (its growth is a one-off, not a per-step cost)
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

    # max over ranks
    tm = torch.tensor([ms, e2e_ms, eval_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ms, e2e_ms, eval_ms = tm.tolist()
    ms_step = ms / args.steps
    units = cfg.gates * Wr * world
    value = units / (ms_step / 1e3)
    e2e_value = units / (e2e_ms / 1e3)

    # roofline of K4 (this rank's work; identical every step).  Toggle totals
    # come from this rank's own per-net counts: n_in = sum over pins of the
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
            pj = json.load(open(prof))
            for ent in (pj if isinstance(pj, list) else [pj]):
                if ent.get("config") == cfg.name and ent.get("windows") == Wr:
                    traffic = ent.get("dram_bytes_per_launch")
        except Exception:
            pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sample = args.cpu_windows or 2048
        r, dt = cpu_oracle_rate(cfg, model, sample, threads)
        cpu = {"value": r, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{cfg.name} design, windows [0,{sample}) in chunks of 256: oracle "
                         f"port (reference algorithm) count+store passes + dwell on {threads} "
                         f"host threads, {dt:.1f} s of CPU work"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "int64", "data": "synthetic (counter-based RNG stimulus, random-init "
                                          "design of the config's shape)",
                "config": {**config_desc(cfg, Wr), "parallelism": f"windows sharded x{world}"},
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
                "activity": {"input_toggles_per_gw": in_tog / (cfg.gates * Wr),
                             "output_toggles_per_gw": out_tog / (cfg.gates * Wr),
                             "chunks_per_step": timing["chunks"]}}
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
