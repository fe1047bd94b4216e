#!/usr/bin/env python
"""Benchmark of the fixed fan-in sparse output layer (arXiv 2306.03725) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--shape S]

A "step" is one training step of the hot path on one synthetic batch (B = 32):
the fused forward / BCE gradient / dW / db / dh / Adam kernel (+ its h-transpose and dh
epilogue kernels), with the SET redistribution run inside the timed region whenever the
global step count reaches a multiple of 1000 — so it is amortised exactly as in
training.  Inference (top-K prediction, row a8) is timed in the same run ("predict").

N = 1 runs in-process; N > 1 is launched by torchrun (one rank per GPU, NCCL): each rank
owns a contiguous label shard, h is broadcast from rank 0 and dh is all-reduced every
step (strong scaling of a fixed global batch).  Rank 0 prints one JSON line.

--impl reference times the fp64 CPU oracle (the reference arm of this tier) on a
bounded sample of the same workload; rank 0 only.
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

METRIC = "train samples/sec & HBM GB/s fraction, Amazon-670K shape, 1/2/4/8 B200"
REDIST_EVERY = 1000          # P:683 "Every 1000 training steps"
PROF_EVERY = 8               # row-kernel launches timed by CUDA events on every 8th timed step
N_BATCHES = 8                # distinct synthetic batches cycled through
LR = 1e-3                    # P:678 initial learning rate


def args_():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--shape", default="amazon-670k")
    p.add_argument("--batch", type=int, default=0,
                   help="override the shape's mini-batch B (default: the paper's 32, P:685); for batch sweeps")
    p.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps")
    p.add_argument("--repeats", type=int, default=5,
                   help="timed windows of --steps steps each; the median window is reported (SURVEY §8(d).3)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--train-only", action="store_true",
                   help="dev A/B sweeps: time the training windows only (no e2e / predict / model / extra sections)")
    p.add_argument("--flags", type=int, default=0, help="extra ff_config.flags (A/B experiments)")
    p.add_argument("--loss", default="bce", choices=["bce", "sqh"],
                   help="bce (north star) or the paper's squared hinge with implicit negative mining (P:526-551)")
    p.add_argument("--margin-bias", type=float, default=0.0,
                   help="sqh: start every label bias at -X so that a controlled fraction of negatives meets the "
                        "margin (engineered-margin analog of a trained model, SURVEY §8(f) NEXT-1)")
    p.add_argument("--hybrid-frac", type=float, default=0.0,
                   help="--dh-mode hybrid: fraction of the columns reduced by red (0 -> library default 0.5)")
    p.add_argument("--dh-mode", default=None, choices=["atomic", "csc", "hybrid"],
                   help="dh scatter: the deterministic CSC pull or red.global atomics; default: the mode measured "
                        "faster for the loss (DESIGN.md §6) — CSC for BCE (1.3-1.5%% faster since the row pass "
                        "gathers into registers), atomic for the squared hinge (its skipped reductions)")
    a = p.parse_args()
    if a.dh_mode is None:                       # the mode measured faster for this loss
        a.dh_mode = "atomic" if a.loss == "sqh" else "csc"
    return a


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(key):
    """dram bytes per launch of `key` from the committed ncu --set full summary, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(key)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], [], set()
        for ln in (self.out or "").splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# measured ceilings of the step's on-chip pattern (tools/microbench/l2bench.cu, profiles/r01_l2bench.txt and
# r01b_l2bench_bulkred.txt): 21.4 M random 128-B line gathers + 21.4 M 128-B red.v4 lines = 11.2 TB/s combined
# (atomic dh); two gathers per connection (CSC pull) ~19.9 TB/s
ONCHIP_CEILING_GBS = {"atomic": 11200.0, "csc": 19900.0}
GATHER_CEILING_GBS = 19900.0      # random 128-B line gathers from an L2-resident table (r01_l2bench)


def gather_bytes(shape, B):
    """On-chip bytes a forward/predict pass gathers: one 128-B h line per connection and
    32-sample chunk (samples padded to whole lines)."""
    return 128.0 * shape.L * shape.k * ((B + 31) // 32)


# ----------------------------------------------------------------------------- byte models
def alg_bytes_train_kernel(L, k):
    """Algorithmic HBM bytes of one fused-step kernel launch:
    read W, idx, mW, vW and write W, mW, vW (28 B per connection); read+write bias, mb, vb
    (24 B per label)."""
    return 28 * L * k + 24 * L


def alg_bytes_step(L, k, B, m, nnz):
    """Algorithmic HBM bytes of one whole step: the kernel's state traffic + read h and
    write dh (8 B per h element) + the labels, + the redistribution amortised over 1000
    steps (read W, idx, mW, vW; write <= 4 arrays in the pruned slots ~ 0.024 L k)."""
    return alg_bytes_train_kernel(L, k) + 8 * B * m + 4 * (B + 1 + nnz) + 0.024 * L * k


def alg_bytes_predict(L, k, B, m):
    return 8 * L * k + 4 * L + 4 * B * m


# ----------------------------------------------------------------------------- cpu baseline
def host_cores():
    return len(os.sched_getaffinity(0))


def oracle_timed(shape, data, steps, warmup, step_budget_s):
    """Time the fp64 oracle as it stands, in its OpenMP timing mode on every host core
    (SURVEY §8(d).4), for `steps` steps after `warmup` untimed ones.  Each step runs the
    full label count when one full step fits `step_budget_s`, else the first `rows` label
    rows (a bounded sample; rows chosen from a probe step on L/32 rows).  Returns
    (rows, measured seconds per step of what ran, threads)."""
    import oracle
    oracle.build()
    cores = host_cores()
    oracle.set_threads(cores)
    try:
        probe = max(1, shape.L // 32)
        st = oracle.State.create(probe, shape.m, shape.k, seed=42)
        t0 = time.perf_counter()
        h, ptr, ids = data[0]
        oracle.train_step(st, h, ptr, ids, 1.0 / shape.B, LR)
        t_full = (time.perf_counter() - t0) * shape.L / probe
        rows = shape.L if t_full <= step_budget_s else max(1, int(shape.L * step_budget_s / t_full))
        st = oracle.State.create(rows, shape.m, shape.k, seed=42)
        for s in range(warmup):
            h, ptr, ids = data[s % len(data)]
            oracle.train_step(st, h, ptr, ids, 1.0 / shape.B, LR)
        t0 = time.perf_counter()
        for s in range(steps):
            h, ptr, ids = data[(warmup + s) % len(data)]
            oracle.train_step(st, h, ptr, ids, 1.0 / shape.B, LR)
        dt = (time.perf_counter() - t0) / max(steps, 1)
    finally:
        oracle.set_threads(1)
    return rows, dt, cores


def cpu_line(shape, rows, dt, cores, steps, warmup):
    """The measured oracle numbers: ms per step of what ran; samples/s of the workload (the
    full label count, so a sampled run's rate is scaled by L / rows and says so)."""
    full = rows == shape.L
    value = shape.B / (dt * shape.L / rows)
    sample = (f"{'all' if full else f'first {rows} of'} {shape.L} label rows, m={shape.m}, k={shape.k}, "
              f"B={shape.B}; fp64 oracle (OpenMP timing mode, {cores} threads), {warmup} warm-up + {steps} timed "
              f"steps of {dt * 1e3:.1f} ms each" + ("" if full else f", rate scaled x{shape.L / rows:.2f} to all rows"))
    out = {"value": value, "unit": "samples/s", "cores": cores, "kind": "oracle", "sample": sample,
           "rows_per_step": rows, "ms_per_step_measured": dt * 1e3}
    if not full:
        out["extrapolated_full_L"] = {"ms_per_step": dt * 1e3 * shape.L / rows, "value": value}
    return out


def run_reference(a, shape, world, rank):
    """This tier's reference arm: the fp64 CPU oracle, on rank 0 only (other ranks exit)."""
    if rank != 0:
        return
    from paper_2306_03725_b200 import synth
    data = [(synth.hidden_batch(shape.B, shape.m, step=s), *synth.label_batch(shape.B, shape.L, shape.avg_pos, step=s))
            for s in range(N_BATCHES)]
    # the whole --steps K --warmup W run is bounded to ~150 s of oracle work
    budget = 150.0 / max(1, a.steps + a.warmup)
    rows, dt, cores = oracle_timed(shape, data, a.steps, a.warmup, budget)
    cb = cpu_line(shape, rows, dt, cores, a.steps, a.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "samples/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: h = ReLU(N(0,1)), Zipf(1.0) sparse labels, Philox-initialized W/idx (no dataset)",
            "config": {"workload": shape.name, "L": shape.L, "m": shape.m, "k": shape.k, "B": shape.B,
                       "rows_per_step": rows},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if rows < shape.L:
        line["extrapolated_full_L"] = cb["extrapolated_full_L"]
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- NEXT-2


def run_sqh(shape, dev, stream, e0, e1, h_dev, ptr_dev, ids_dev, margin=3.0, steps=300):
    """the paper's squared-hinge loss with implicit negative mining
     on the same batches, the label biases set to -margin so that almost every
    (sample, label) gradient is exactly zero (engineered margins, SURVEY d.1); samples/s and
    the fraction of exact-zero gradients on the first batch."""
    import torch
    from paper_2306_03725_b200 import synth
    from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig, FF_LOSS_SQH
    B = shape.B
    lay = FixedFanInLayer(LayerConfig(L_global=shape.L, m=shape.m, k=shape.k, max_batch=B, seed=synth.PARAM_SEED,
                                      loss=FF_LOSS_SQH), device=dev)
    lay.set_params(bias=torch.full((shape.L,), -margin, dtype=torch.float32, device=dev))
    y = lay.forward(h_dev[0])
    t = -torch.ones_like(y)
    p_, i_ = ptr_dev[0].cpu().numpy(), ids_dev[0].cpu().numpy()
    for b in range(B):
        t[b, torch.from_numpy(i_[p_[b]:p_[b + 1]].astype(np.int64)).to(dev)] = 1.0
    skip = float(((t * y) >= 1.0).float().mean().item())
    del y, t
    dh = torch.empty((B, shape.m), device=dev)
    n = len(h_dev)
    for s in range(20):
        lay.train_step(h_dev[s % n], ptr_dev[s % n], ids_dev[s % n], LR, dh=dh)
    torch.cuda.synchronize()
    e0.record(stream)
    for s in range(steps):
        lay.train_step(h_dev[s % n], ptr_dev[s % n], ids_dev[s % n], LR, dh=dh)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    del lay
    return {"loss": "squared hinge (P:526-529)", "margin_bias": margin, "grad_skip_fraction": skip,
            "value": B / (ms * 1e-3), "unit": "samples/s", "ms_per_step": ms, "steps": steps}


def run_model(eng, shape, dev, stream, e0, e1, d=512, dropout=0.1, steps=100):
    """the whole proposed architecture (Fig. 2): 512-d Slice-like features
     -> 10% input dropout -> dense Wd -> ReLU -> the fixed fan-in layer, one
    fused fixedfanin_model_train_step per batch; plus the two dense kernels timed alone."""
    import torch
    from paper_2306_03725_b200 import synth
    from paper_2306_03725_b200.layer import DenseConfig, DenseLayer, last_launch_count, model_train_step
    B = shape.B
    dn = DenseLayer(DenseConfig(d=d, m=shape.m, max_batch=B, seed=synth.PARAM_SEED + 1, dropout=dropout), device=dev)
    xs = [torch.from_numpy(synth.feature_batch(B, d, step=s)).to(dev) for s in range(N_BATCHES)]
    lbl = [(torch.from_numpy(p).to(dev), torch.from_numpy(i).to(dev))
           for p, i in (synth.label_batch(B, shape.L, shape.avg_pos, step=s) for s in range(N_BATCHES))]
    loss = torch.zeros(1, device=dev)
    for s in range(3):
        model_train_step(dn, eng, xs[s % N_BATCHES], s, *lbl[s % N_BATCHES], LR, loss=loss)
    launches = last_launch_count()
    e0.record(stream)
    for s in range(steps):
        model_train_step(dn, eng, xs[s % N_BATCHES], s, *lbl[s % N_BATCHES], LR, loss=loss)
    e1.record(stream)
    e1.synchronize()
    ms_model = e0.elapsed_time(e1) / steps
    h = torch.empty((B, shape.m), device=dev)
    dh = torch.from_numpy(synth.hidden_batch(B, shape.m, step=5) * np.float32(1e-3)).to(dev)
    res = {}
    # the dense kernels alone, timed as CUDA-graph replays of 20 calls (a Python loop of these
    # calls is host-bound at ~20 us per call, longer than the forward itself)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for name, fn in (("fwd", lambda: dn.forward(xs[0], step=1, train=True, h=h)),
                         ("bwd", lambda: (dn.forward(xs[0], step=1, train=True, h=h), dn.backward_adam(dh, LR)))):
            fn()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                for _ in range(20):
                    fn()
            g.replay()
            e0.record(side)
            for _ in range(5):
                g.replay()
            e1.record(side)
            e1.synchronize()
            res[name] = e0.elapsed_time(e1) / 100
            del g
    torch.cuda.current_stream().wait_stream(side)
    res["bwd"] -= res["fwd"]
    peak, peak_src = peaks()
    bwd_bytes = 24 * d * shape.m + 8 * d * 32 + 8 * shape.m * 32 + 4 * B * shape.m
    fwd_flops = 2 * B * d * shape.m
    fwd_bytes = 4 * d * shape.m + 8 * 32 * shape.m
    del dn
    return {"workload": f"{shape.name} + dense intermediate d={d}, dropout {dropout}", "d": d, "B": B,
            "value": B / (ms_model * 1e-3), "unit": "samples/s", "ms_per_step": ms_model,
            "launches_per_step": launches,
            "dense_fwd": {"ms": res["fwd"], "bound": "hbm", "alg_bytes": fwd_bytes,
                          "achieved_gbs": fwd_bytes / (res["fwd"] * 1e-3) / 1e9, "peak_gbs": peak,
                          "frac": fwd_bytes / (res["fwd"] * 1e-3) / 1e9 / peak,
                          "tflops_3xtf32": 3 * fwd_flops / (res["fwd"] * 1e-3) / 1e12,
                          "note": "CUDA-graph replay: dropout kernel + k_dense_fwd_tma (TMA-fed tcgen05 kind::tf32 3xTF32, "
                                  "M = 128 columns, N = 64 [x_hi | x_lo] + N = 32, bias/ReLU epilogue from TMEM); "
                                  "bytes = read Wd + write the h|dh lines; bound by shared-memory bandwidth "
                                  "(DESIGN.md 6c)"},
            "dense_bwd_adam": {"ms": res["bwd"], "bound": "hbm", "alg_bytes": bwd_bytes,
                               "achieved_gbs": bwd_bytes / (res["bwd"] * 1e-3) / 1e9, "peak_gbs": peak,
                               "peak_source": peak_src, "frac": bwd_bytes / (res["bwd"] * 1e-3) / 1e9 / peak,
                               "note": "dh transpose-in + dWd = xt^T dz fused with Adam over Wd/mWd/vWd "
                                       "(24 B per weight)"}}


# ----------------------------------------------------------------------------- ours
def run_ours(a, shape, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2306_03725_b200 import synth
    from paper_2306_03725_b200.layer import last_launch_count
    from paper_2306_03725_b200.sharded import ShardedLayer

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    B = shape.B
    data = [(synth.hidden_batch(B, shape.m, step=s), *synth.label_batch(B, shape.L, shape.avg_pos, step=s))
            for s in range(N_BATCHES)]
    max_nnz = max(int(d[1][-1]) for d in data)
    from paper_2306_03725_b200.layer import FF_DH_ATOMIC, FF_DH_CSC, FF_LOSS_BCE, FF_LOSS_SQH
    from paper_2306_03725_b200.layer import FF_DH_HYBRID
    dh_mode = {"csc": FF_DH_CSC, "hybrid": FF_DH_HYBRID}.get(a.dh_mode, FF_DH_ATOMIC)
    layer = ShardedLayer(shape.L, shape.m, shape.k, rank=rank, world=world, device=dev, max_batch=B,
                         seed=synth.PARAM_SEED, max_nnz=max_nnz, dh_mode=dh_mode, flags=a.flags,
                         loss=FF_LOSS_SQH if a.loss == "sqh" else FF_LOSS_BCE, hybrid_frac=a.hybrid_frac)
    eng = layer.engine
    L_local = layer.row_end - layer.row_begin
    stream = torch.cuda.current_stream()

    h_dev = [torch.from_numpy(d[0]).to(dev) for d in data]
    ptr_dev = [torch.from_numpy(d[1]).to(dev) for d in data]
    ids_dev = [torch.from_numpy(d[2]).to(dev) for d in data]
    skip_fraction = None
    if a.margin_bias:
        eng.set_params(bias=torch.full((L_local,), -a.margin_bias, dtype=torch.float32, device=dev))
    if a.loss == "sqh":
        # fraction of (sample, label) gradients that are exactly zero on the first batch (t' y >= 1)
        y = eng.forward(h_dev[0])
        t = -torch.ones_like(y)
        p_, i_ = data[0][1], data[0][2]
        for b in range(B):
            loc = [int(x) - layer.row_begin for x in i_[p_[b]:p_[b + 1]] if layer.row_begin <= x < layer.row_end]
            if loc:
                t[b, loc] = 1.0
        skip_fraction = float(((t * y) >= 1.0).float().mean().item())
        del y, t
    dh = torch.empty((B, shape.m), device=dev)
    loss = torch.zeros(1, device=dev)
    t_global = 0
    launches = 0

    from paper_2306_03725_b200.sharded import OverlappedTrainer
    trainer = OverlappedTrainer(layer, h_dev, ptr_dev, ids_dev, LR, B, shape.m, dev, loss=loss)

    n_redist = 0

    def step(s):
        nonlocal t_global, launches, n_redist
        trainer.step(s % N_BATCHES, (s + 1) % N_BATCHES)     # h broadcast / dh all-reduce overlapped
        launches += last_launch_count()
        t_global += 1
        if t_global % REDIST_EVERY == 0:
            layer.redistribute(t_global)
            launches += last_launch_count()
            n_redist += 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for s in range(a.warmup):
        step(s)
    trainer.finish()
    barrier()
    # The global step counter drives the redistribution cadence ("every 1000 training
    # steps").  A window of K >= 1000 steps crosses its multiples naturally; a shorter window
    # is placed so that it crosses exactly one (t_global starts K/2 before a multiple of
    # 1000): such a window then carries one redistribution per K steps, more than the
    # amortised 1/1000 (conservative; `redistribution` reports the amortised share).
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    windows, own_windows, host_ms, redist_per_window, launch_counts = [], [], [], [], []
    k_ms_tot, k_n_tot, n_prof = 0.0, 0, 0
    samplers = []
    for rep in range(max(1, a.repeats)):
        if a.steps < REDIST_EVERY:
            t_global = REDIST_EVERY * (rep + 1) - a.steps // 2
        launches, n_redist = 0, 0
        # the row kernel is timed by CUDA events around its launches on every PROF_EVERY-th step
        # of the timed loop (each event pair costs the step ~6 us; tools/prof_overhead.py)
        eng.profile_begin(a.steps * 16)
        sampler = ClockSampler(local_rank)
        with sampler:
            barrier()
            e0.record(stream)
            t_h0 = time.perf_counter()
            for s in range(a.steps):
                if PROF_EVERY > 1:
                    eng.profile_pause(s % PROF_EVERY != 0)
                step(a.warmup + s)
            trainer.finish()                                     # every collective inside the timed region
            host_ms.append((time.perf_counter() - t_h0) * 1e3 / a.steps)   # enqueue time (no sync yet)
            e1.record(stream)
            barrier()
        own_windows.append(e0.elapsed_time(e1))
        windows.append(max_over_ranks(own_windows[-1]))
        k_ms, k_n = eng.profile_end()
        k_ms_tot += k_ms; k_n_tot += k_n; n_prof += len(range(0, a.steps, PROF_EVERY))
        redist_per_window.append(n_redist)
        launch_counts.append(launches)
        samplers.append(sampler)
    med = sorted(range(len(windows)), key=lambda i: windows[i])[len(windows) // 2]
    clk = samplers[med]                                   # clocks of the reported window
    ms = windows[med]
    k_step_ms = max_over_ranks(k_ms_tot / n_prof)        # fused row kernel time per step (all its launches)
    launches_per_step = k_n_tot / n_prof
    gpu_launches = launch_counts[med]

    # ---- N > 1: where a rank's step goes: the same steps with the shard's
    # compute only (no collectives) and the collectives only (h broadcast + dh all-reduce),
    # each timed on this rank's stream; gathered to rank 0
    per_rank = None
    if world > 1:
        def timed(fn):
            barrier()
            e0.record(stream)
            for s in range(a.steps):
                fn(s)
            e1.record(stream)
            barrier()
            return e0.elapsed_time(e1) / a.steps
        compute_ms = timed(lambda s: eng.train_step(h_dev[s % N_BATCHES], ptr_dev[s % N_BATCHES], ids_dev[s % N_BATCHES],
                                                    LR, dh=dh, loss=loss))
        comm_ms = timed(lambda s: (dist.broadcast(h_dev[s % N_BATCHES], src=0), dist.all_reduce(dh)))
        rec = {"rank": rank, "L_local": L_local, "step_ms": own_windows[med] / a.steps,
               "row_kernel_ms": k_ms_tot / n_prof, "compute_only_ms": compute_ms, "comm_only_ms": comm_ms,
               "exposed_comm_ms": own_windows[med] / a.steps - compute_ms, "host_enqueue_ms": host_ms[med]}
        per_rank = [None] * world
        dist.all_gather_object(per_rank, rec)
    if a.train_only:
        if rank == 0:
            print(json.dumps({"ms_per_step": ms / a.steps, "value": B * a.steps / (ms * 1e-3),
                              "windows_ms_per_step": [w / a.steps for w in windows],
                              "row_kernel_ms_per_step": k_step_ms, "row_launches_per_step": launches_per_step,
                              "dh_mode": a.dh_mode, "loss": a.loss, "B": B, "shape": shape.name}), flush=True)
        return
    # ---- end to end through the public API with host buffers (H2D inputs, D2H loss)
    n_e2e = a.e2e_steps or a.steps
    h_pin = [torch.from_numpy(d[0]).pin_memory() for d in data]
    ptr_pin = [torch.from_numpy(d[1]).pin_memory() for d in data]
    ids_pin = [torch.from_numpy(d[2]).pin_memory() for d in data]
    loss_pin = torch.zeros(1).pin_memory()
    h2d = B * shape.m * 4 + int(np.mean([4 * (B + 1 + len(d[2])) for d in data]))
    d2h = 4
    dh_pin = torch.empty((B, shape.m)).pin_memory()
    want_dh = False                       # second e2e pass: the step's [B][m] dh output comes back too

    def step_e2e(s):
        nonlocal t_global
        i = s % N_BATCHES
        if world == 1:
            eng.train_step_host(h_pin[i], ptr_pin[i], ids_pin[i], LR, loss_host=loss_pin,
                                dh_host=dh_pin if want_dh else None)
        else:
            # the producer rank's h reaches the device by H2D and the other ranks by the
            # broadcast inside trainer.step; every rank copies its labels; the dh all-reduce of
            # this step overlaps the next step (OverlappedTrainer)
            if rank == 0:
                h_dev[i].copy_(h_pin[i], non_blocking=True)
            ptr_dev[i].copy_(ptr_pin[i], non_blocking=True)
            ids_dev[i].copy_(ids_pin[i], non_blocking=True)
            dh_s = trainer.step(i, None)
            loss_pin.copy_(loss, non_blocking=True)
            if want_dh:
                trainer.finish()
                dh_pin.copy_(dh_s, non_blocking=True)
        t_global += 1
        if t_global % REDIST_EVERY == 0:
            layer.redistribute(t_global)

    for s in range(3):
        step_e2e(s)
    trainer.finish()
    with ClockSampler(local_rank) as clk2:
        barrier()
        e0.record(stream)
        for s in range(n_e2e):
            step_e2e(s)
        trainer.finish()
        e1.record(stream)
        barrier()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1))
    want_dh = True
    for s in range(3):
        step_e2e(s)
    barrier()
    e0.record(stream)
    for s in range(n_e2e):
        step_e2e(s)
    trainer.finish()
    e1.record(stream)
    barrier()
    ms_e2e_dh = max_over_ranks(e0.elapsed_time(e1))

    # ---- inference: fused forward + top-K (row a8), K = 5 (P@1/3/5)
    K = 5
    for s in range(3):
        layer.predict_topk(h_dev[s % N_BATCHES], K)
    n_pred = 100
    barrier()
    e0.record(stream)
    for s in range(n_pred):
        layer.predict_topk(h_dev[s % N_BATCHES], K)
    e1.record(stream)
    barrier()
    ms_pred = max_over_ranks(e0.elapsed_time(e1))

    # ---- row a7 on its own: one redistribution (prune + Philox regrow + moment reset, and the
    # CSC rebuild in csc/hybrid mode), which the timed train loop amortises over 1000 steps.
    # Algorithmic bytes: read W and idx (8 B per connection) + write idx, W, mW, vW of the
    # p = floor(0.1 k) regrown slots per row (16 B each).
    n_red = 5
    layer.redistribute(10 ** 6)
    barrier()
    e0.record(stream)
    for r in range(n_red):
        layer.redistribute(10 ** 6 + 1000 * (r + 1))
    e1.record(stream)
    barrier()
    ms_red = max_over_ranks(e0.elapsed_time(e1)) / n_red
    p_slots = (shape.k * 10) // 100
    red_bytes = 8.0 * L_local * shape.k + 16.0 * L_local * p_slots
    redist = {"ms_per_call": ms_red, "amortised_ms_per_step": ms_red / REDIST_EVERY,
              "share_of_step": ms_red / REDIST_EVERY / (ms / a.steps),
              "alg_bytes": red_bytes, "achieved_gbs": red_bytes / (ms_red * 1e-3) / 1e9,
              "frac": red_bytes / (ms_red * 1e-3) / 1e9 / peaks()[0],
              "note": "prune p = floor(0.1 k) smallest |W| per row, regrow by Philox (seed, step, row)"
                      + ("; includes the CSC rebuild" if a.dh_mode != "atomic" else "")}

    # ---- the same training step captured once in a CUDA graph and replayed (static input
    # buffers; the device-side Adam counter advances per replay): host launch cost per step
    # drops to one graph launch
    graph = None
    if world == 1:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            layer.train_step(h_dev[0], ptr_dev[0], ids_dev[0], LR, dh=dh, loss=loss)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            layer.train_step(h_dev[0], ptr_dev[0], ids_dev[0], LR, dh=dh, loss=loss)
        n_g = 200
        for _ in range(3):
            g.replay()
        barrier()
        e0.record(stream)
        for _ in range(n_g):
            g.replay()
        e1.record(stream)
        barrier()
        ms_g = e0.elapsed_time(e1) / n_g
        graph = {"ms_per_step": ms_g, "samples_per_s": B / (ms_g * 1e-3), "steps": n_g,
                 "note": "one captured fixedfanin_train_step replayed on static buffers (redistribution not included)"}
        del g
    elif dist.get_backend() == "nccl":
        # N > 1: the sharded steps WITH their collectives in one graph (sharded.GraphedSteps:
        # per step the h broadcast, the shard's fused step and the async dh all-reduce, which
        # overlaps the next step inside the graph); NCCL collectives are capturable, gloo's not
        from paper_2306_03725_b200.sharded import GraphedSteps
        gs = GraphedSteps(layer, h_dev, ptr_dev, ids_dev, LR, B, shape.m, dev, loss=loss)
        n_rep = max(1, 200 // gs.K)
        for _ in range(2):
            gs.replay()
        barrier()
        e0.record(stream)
        for _ in range(n_rep):
            gs.replay()
        e1.record(stream)
        barrier()
        ms_g = max_over_ranks(e0.elapsed_time(e1) / (n_rep * gs.K))
        graph = {"ms_per_step": ms_g, "samples_per_s": B / (ms_g * 1e-3), "steps": n_rep * gs.K,
                 "steps_per_graph": gs.K,
                 "note": "sharded.GraphedSteps: K steps (h broadcast + fused step + async dh all-reduce each) per "
                         "captured graph, max over ranks (redistribution not included)"}
        del gs

    # ---- NEXT-3: large-batch inference and shortlist scoring, one GPU
    big = model = sqh = None
    if world == 1:
        from paper_2306_03725_b200.layer import FixedFanInLayer, LayerConfig
        BI, NCAND = 1024, 100
        inf = FixedFanInLayer(LayerConfig(L_global=shape.L, m=shape.m, k=shape.k, max_batch=BI,
                                          seed=synth.PARAM_SEED), device=dev)
        inf.set_params(**{key: v for key, v in eng.get_params().items() if torch.is_tensor(v)})
        hb = torch.from_numpy(synth.hidden_batch(BI, shape.m, step=99)).to(dev)
        rng = np.random.default_rng(7)
        cptr = torch.arange(BI + 1, dtype=torch.int32, device=dev) * NCAND
        cids = torch.from_numpy(rng.integers(0, shape.L, size=BI * NCAND).astype(np.int32)).to(dev)
        scores = torch.empty(BI * NCAND, dtype=torch.float32, device=dev)
        res = {}
        for name, fn, reps in (("predict", lambda: inf.predict_topk(hb, K), 5),
                               ("shortlist", lambda: inf.score_shortlist(hb, cptr, cids, scores), 50)):
            fn()
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            e1.synchronize()
            res[name] = e0.elapsed_time(e1) / reps
        big = {"B": BI, "K": K, "predict_samples_per_s": BI / (res["predict"] * 1e-3),
               "predict_ms_per_batch": res["predict"],
               "predict_gather_floor_ms": gather_bytes(shape, BI) / (GATHER_CEILING_GBS * 1e9) * 1e3,
               "predict_gather_frac": gather_bytes(shape, BI) / (res["predict"] * 1e-3) / 1e9 / GATHER_CEILING_GBS,
               "shortlist_candidates_per_sample": NCAND, "shortlist_pairs_per_s": BI * NCAND / (res["shortlist"] * 1e-3),
               "shortlist_ms_per_batch": res["shortlist"]}
        del inf
        model = run_model(eng, shape, dev, stream, e0, e1)
        if a.loss == "bce" and not a.train_only:
            sqh = run_sqh(shape, dev, stream, e0, e1, h_dev, ptr_dev, ids_dev)

    if rank != 0:
        return
    peak, peak_src = peaks()
    samples_per_s = B * a.steps / (ms * 1e-3)
    kb = alg_bytes_train_kernel(L_local, shape.k)        # per step = per launch x launches_per_step
    achieved = kb / (k_step_ms * 1e-3) / 1e9
    nnz_mean = float(np.mean([len(d[2]) for d in data]))
    step_bytes = alg_bytes_step(shape.L, shape.k, B, shape.m, nnz_mean)
    traffic = ncu_traffic(f"{shape.name}/{a.dh_mode}/train_kernel")
    nbl = (B + 31) // 32
    onchip = 2 * 128 * L_local * shape.k * nbl   # h line gathers + dh line reductions (atomic) or g line gathers (CSC)
    # what the timed (row) kernel itself moves on chip: atomic = h gathers + dh reds per connection;
    # CSC row pass = h gathers per connection + the row's g line and W line (the column pass,
    # k_dh_csc, gathers the g lines and is not inside the timed row-kernel launches)
    onchip_kernel = onchip if a.dh_mode == "atomic" else (128 * L_local * shape.k + 256 * L_local) * nbl
    pred_bytes = alg_bytes_predict(shape.L, shape.k, B, shape.m)
    c1, c2 = clk.summary(), clk2.summary()
    line = {
        "metric": METRIC, "value": samples_per_s, "unit": "samples/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: h = ReLU(N(0,1)), Zipf(1.0) sparse labels, Philox-initialized W/idx (no dataset)",
        "config": {"workload": shape.name, "L": shape.L, "m": shape.m, "k": shape.k, "B": B, "global_batch": B,
                   "avg_pos": shape.avg_pos, "parallelism": f"label-shard x{world}", "dh_mode": a.dh_mode,
                   "hybrid_frac": (a.hybrid_frac or 0.5) if a.dh_mode == "hybrid" else None,
                   "loss": a.loss, "margin_bias": a.margin_bias, "grad_skip_fraction": skip_fraction,
                   "redistribution": (f"at every multiple of {REDIST_EVERY} of the global step counter; "
                                      f"{redist_per_window[med]} inside the reported window of {a.steps} steps"
                                      + (" (window placed to cross one multiple)" if a.steps < REDIST_EVERY else "")),
                   "l2": "no flush: per-step state stream 617 MB >> 126 MB L2 (inputs larger than L2)"},
        "repeats": {"windows_ms_per_step": [w / a.steps for w in windows], "reported": "median",
                    "redistributions_per_window": redist_per_window},
        "clocks": {"sm_mhz": c1["sm_mhz"], "sm_max_mhz": c1["sm_max_mhz"], "reasons": c1["reasons"],
                   "samples": c1["samples"]},
        "hbm_step": {"alg_bytes_per_step": step_bytes, "achieved_gbs": step_bytes / (ms / a.steps * 1e-3) / 1e9,
                     "frac": step_bytes / (ms / a.steps * 1e-3) / 1e9 / peak},
        "e2e": {"value": B * n_e2e / (ms_e2e * 1e-3), "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": n_e2e, "ms_per_step": ms_e2e / n_e2e,
                "path": "fixedfanin_train_step_host (C ABI, pinned host buffers)" if world == 1 else
                        "torch H2D (h on the producer rank, labels on every rank) + OverlappedTrainer step "
                        "(h broadcast, fused step, dh all-reduce overlapped with the next step) + D2H loss",
                "clocks_sm_mhz": c2["sm_mhz"]},
        "e2e_with_dh": {"value": B * n_e2e / (ms_e2e_dh * 1e-3), "unit": "samples/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h + 4 * B * shape.m, "steps": n_e2e,
                        "ms_per_step": ms_e2e_dh / n_e2e,
                        "note": "as e2e, plus the step's dh [B][m] copied back to pinned host memory every step"},
        "gpu_launches": gpu_launches,
        # `bound` names the roof the ncu evidence shows binding (profiles/r01d_ncu_train_ring_atomic.txt:
        # L1->XBAR request path ~89% busy, DRAM ~13%); achieved / peak / frac stay the north star's
        # HBM fraction (algorithmic bytes), and `binding` relates the same launch to its on-chip roof.
        "roofline": {"bound": "l2", "kernel": ("k_train_ring (fused fwd/BCE/dW/db/dh-or-g/Adam row pass)"
                                                 + ("; CSC: one launch per label tile, each followed by the column "
                                                    "pass k_dh_csc (in the step time, not in this kernel's)"
                                                    if a.dh_mode == "csc" else "")),
                     "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": achieved / peak, "hbm_frac": achieved / peak, "traffic": traffic,
                     "binding": {"roof": ("L2 gather + reduction path (random 128-B lines)" if a.dh_mode == "atomic"
                                          else "L2 gather path (random 128-B h lines; row pass)"),
                                 "achieved_gbs": onchip_kernel / (k_step_ms * 1e-3) / 1e9,
                                 "ceiling_gbs": ONCHIP_CEILING_GBS.get(a.dh_mode),
                                 "frac": (onchip_kernel / (k_step_ms * 1e-3) / 1e9 / ONCHIP_CEILING_GBS[a.dh_mode]
                                          if a.dh_mode in ONCHIP_CEILING_GBS else None)},
                     "alg_bytes_per_launch": kb / launches_per_step, "launches_per_step": launches_per_step,
                     "avg_launch_ms": k_step_ms / launches_per_step,
                     "kernel_share_of_step": k_step_ms / (ms / a.steps),
                     "timing": f"CUDA events around each launch on the launching stream, every {PROF_EVERY}th timed step "
                               f"({n_prof} of {a.steps * max(1, a.repeats)} over {max(1, a.repeats)} windows)"},
        # SURVEY §8(d).2's third ceiling: FP32 issue.  3 B L k FMAs per step (forward, dW, dh
        # contributions) in the row kernel against 148 SMs x 128 FP32 lanes x the max SM clock
        # (FFMA2 issues two lanes' worth per instruction; nominal ~74 TFLOP/s)
        "fp32": {"fma_per_step": 3.0 * B * L_local * shape.k,
                 "kernel_tfma_s": 3.0 * B * L_local * shape.k / (k_step_ms * 1e-3) / 1e12,
                 "peak_tfma_s": 148 * 128 * 1.965e9 / 1e12,
                 "frac": 3.0 * B * L_local * shape.k / (k_step_ms * 1e-3) / (148 * 128 * 1.965e9),
                 "peak_source": "derived: 148 SMs x 128 FP32 FMA lanes x 1965 MHz"},
        "onchip": {"l2_bytes_per_step": onchip, "l2_gbs": onchip / (ms / a.steps * 1e-3) / 1e9,
                   "kernel_bytes_per_step": onchip_kernel,
                   "kernel_gbs": onchip_kernel / (k_step_ms * 1e-3) / 1e9,
                   "ceiling_gbs": ONCHIP_CEILING_GBS.get(a.dh_mode),
                   "kernel_frac_of_ceiling": (onchip_kernel / (k_step_ms * 1e-3) / 1e9 / ONCHIP_CEILING_GBS[a.dh_mode]
                                              if a.dh_mode in ONCHIP_CEILING_GBS else None),
                   # The state stream (W, idx, moments, bias) also passes through the L2 slices: the kernel's
                   # total L2 rate is the gather/red bytes plus its algorithmic HBM bytes over its duration.
                   "kernel_l2_total_gbs": (onchip_kernel + kb) / (k_step_ms * 1e-3) / 1e9,
                   "kernel_l2_total_frac_of_ceiling": ((onchip_kernel + kb) / (k_step_ms * 1e-3) / 1e9
                                                       / ONCHIP_CEILING_GBS[a.dh_mode]
                                                       if a.dh_mode in ONCHIP_CEILING_GBS else None),
                   "note": ("h 128-B line gather + dh 128-B red.v4 per connection" if a.dh_mode == "atomic" else
                            "h 128-B line gather (row pass) + g 128-B line gather (CSC column pass) per connection")
                           + "; measured ceilings (profiles/r01_l2bench.txt): gather ~19.9 TB/s, red ~6.3-6.6 TB/s"},
        "host_enqueue_ms_per_step": host_ms[med],
        "per_rank": per_rank,
        "comm": ({"backend": dist.get_backend(), "comm_nranks": dist.get_world_size(),
                  "collectives_per_step": "broadcast h (4 B m) + all_reduce dh (4 B m), overlapped with the next "
                                          "step (OverlappedTrainer)",
                  "nccl_debug": os.environ.get("NCCL_DEBUG")} if world > 1 else None),
        "predict": {"value": B * n_pred / (ms_pred * 1e-3), "unit": "samples/s", "K": K,
                    "ms_per_batch": ms_pred / n_pred,
                    "hbm_gbs": pred_bytes / (ms_pred / n_pred * 1e-3) / 1e9,
                    "frac": pred_bytes / (ms_pred / n_pred * 1e-3) / 1e9 / peak,
                    # the binding roof: the random 128-B h-line gathers (4 B x B_pad x L x k) vs the
                    # measured gather-only ceiling (tools/microbench/l2bench, profiles/r01_l2bench.txt)
                    "gather_gbs": gather_bytes(shape, B) / (ms_pred / n_pred * 1e-3) / 1e9,
                    "gather_floor_ms": gather_bytes(shape, B) / (GATHER_CEILING_GBS * 1e9) * 1e3,
                    "gather_frac": gather_bytes(shape, B) / (ms_pred / n_pred * 1e-3) / 1e9 / GATHER_CEILING_GBS},
        "redistribution": redist,
        "cuda_graph": graph,
        "inference_large_batch": big,
        "model": model if world == 1 else None,
        "sqh": (dict(sqh, ratio_to_bce_step=sqh["ms_per_step"] / (ms / a.steps)) if sqh else None),
    }
    # NEXT-4 memory report: this layer's device bytes vs the dense/COO formats of P:37-45
    Lk = shape.L * shape.k
    line["memory"] = {
        "workspace_bytes_per_gpu": int(eng.workspace.numel()),
        "peak_allocated_bytes": int(torch.cuda.max_memory_allocated(dev)),
        "uniform_params_bytes": 8 * Lk + 4 * shape.L,                 # W + idx (32-bit) + bias
        "uniform_with_adam_bytes": 16 * Lk + 12 * shape.L,            # + mW, vW, mb, vb
        "coo64_params_bytes": 20 * Lk,                                # 2 x int64 + fp32 per nnz
        "dense_params_bytes": 4 * shape.m * shape.L,                  # the dense layer it replaces
        "dense_with_adam_bytes": 12 * shape.m * shape.L,              # weights + two moments
        "note": "dense figures for a dense m x L last layer of the same width (P:37-45 quotes 10.7 GiB "
                "/ >40 GiB for Amazon-3M at 1024 hidden)"}
    if world == 1 and not a.no_cpu_baseline:
        # ~10-30 s of CPU work: 1 warm-up + 3 timed steps, each full-size if it fits 6 s
        rows, dt, cores = oracle_timed(shape, data, 3, 1, 6.0)
        line["cpu_baseline"] = cpu_line(shape, rows, dt, cores, 3, 1)
    print(json.dumps(line), flush=True)


def main():
    a = args_()
    from paper_2306_03725_b200 import synth
    shape = synth.SHAPES[a.shape]
    if a.batch:
        import dataclasses
        shape = dataclasses.replace(shape, B=a.batch)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, shape, world, rank)
        return
    import __graft_entry__
    if world > 1:
        import torch
        import torch.distributed as dist
        # NCCL (one rank per GPU) in production; FF_BENCH_BACKEND=gloo lets several ranks share
        # one GPU to exercise the multi-rank path where only one GPU is available (tests only)
        backend = os.environ.get("FF_BENCH_BACKEND", "nccl")
        gpu = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(gpu)
        if backend == "nccl":
            # NCCL's communicator log (stderr) carries the nranks of every communicator
            if os.environ.get("NCCL_DEBUG", "VERSION").upper() in ("VERSION", "NONE", ""):
                os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
        else:
            dist.init_process_group(backend)
    if rank == 0:
        __graft_entry__.build_lib()          # no-op when the in-tree .so is current
    if world > 1:
        dist.barrier()                       # the other ranks load the library only after rank 0 built it
    run_ours(a, shape, world, rank, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
