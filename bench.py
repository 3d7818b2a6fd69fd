"""PipeOptim hot-path benchmark on B200 — prints ONE JSON line (rank 0).

Workload (a "step"): one fused weight-predict + optimizer-step pass (K3,
Adam, s = 3, t > 0) over one stage's flat fp32 buffers of N = 1e9 parameters
— BASELINE.json configs[4] at its 1B headline point, the configuration the
north-star kernel target (>= 80% of ~8 TB/s at 1B params) is quoted on.
Inputs (W, G, m, v = 16 GB) are larger than L2 (126 MB) so no flush is
needed between steps.

  value   whole-job algorithmic GB/s: N * 32 B * ranks / step
          time, device-timed with CUDA events, max over ranks.
  e2e     the same metric through the reference-facing host-buffer API
          (HostStreamer: pinned host W and G in, W' and W_hat out, PCIe copies
          inside the timed region; optimizer state device-resident); beside
          it the training-loop setting (gradient in, flag out) and the
          reference's three-call list API on host tensors.
  kernels_1e9  K1 / K2 / K3 x SGDM / Adam / AdamW at the same N.
  roofline  K3's achieved GB/s vs MEASURED_PEAKS.json hbm_gbs; `traffic` is
          ncu's dram bytes per launch from profiles/ when captured.
  cpu_baseline  the reference's algorithm (oracle/c, float64, OpenMP on every
          host core) on a bounded sample, same per-parameter byte accounting.
  pipeline  the first metric clause: 1F1B samples/s on config 1 (4-stage
          3072-1024^3-10 MLP, B=128, Adam), prediction on vs off.

--gpus N (torchrun, one process per GPU): the kernel is per-stage state, so N
ranks are N independent stages ("replicas only", scaling weak); the pipeline
leg then runs the real N-stage NCCL pipeline.

--impl reference: the reference's CPU implementation (the oracle port; the
reference is pure Python and cannot travel) timed on the host cores.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_PARAM = {"sgdm": 24, "adam": 32, "adamw": 32}  # K3, SURVEY.md §8d
METRIC = "weight-predict+step HBM GB/s (fused K3; pipeline samples/sec in `pipeline`)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-params", type=float, default=1e9)
    ap.add_argument("--kind", choices=["sgdm", "adam", "adamw"], default="adam")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--pipeline-batches", type=int, default=64)
    ap.add_argument("--pipeline-timeout", type=float, default=None,
                    help="watchdog on the pipeline leg (default 420 s on 1 GPU, 900 s with more ranks)")
    ap.add_argument("--no-configs", action="store_true", help="skip configs 2-4 in the pipeline leg")
    # test-only: exercise the multi-rank bench on ONE GPU (ranks share the
    # device, gloo transport with host staging); never used for numbers
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--share-gpu", action="store_true")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ---- clocks -------------------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.25)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        loaded = [x for x in sm if smax and x > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- helpers --------------------------------------------------------------------------------


def measured_peak():
    try:
        j = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per K3 launch from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "k3_traffic.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def cpu_baseline(kind: str, budget_s: float = 12.0, n: int = 1 << 26):
    """The reference algorithm (oracle/c float64, OpenMP) on a bounded sample."""
    import numpy as np

    from oracle import c_oracle

    c_oracle.build()
    rng = np.random.default_rng(0)
    w = rng.normal(0, 0.02, n)
    g = rng.normal(0, 1e-2, n)
    m = rng.normal(0, 1e-3, n)
    v = rng.normal(0, 1e-2, n) ** 2
    wh = np.empty(n)
    hp = c_oracle.hp(kind)
    s2 = None if kind == "sgdm" else v
    c_oracle.step_predict(hp, w, g, m, s2, wh, 1e-3, 3e-3, 10)  # warm (page-in)
    times, t_start, t = [], time.perf_counter(), 11
    while time.perf_counter() - t_start < budget_s or len(times) < 3:
        t0 = time.perf_counter()
        c_oracle.step_predict(hp, w, g, m, s2, wh, 1e-3, 3e-3, t)
        times.append(time.perf_counter() - t0)
        t += 1
    per = statistics.median(times)
    return {
        "value": round(BYTES_PER_PARAM[kind] * n / per / 1e9, 2),
        "unit": "GB/s",
        "cores": c_oracle.threads(),
        "kind": "port",
        "sample": (f"oracle/c/optim_oracle.c step+predict ({kind}, float64 like the reference, OpenMP) on "
                   f"{n} params x {len(times)} reps, median {per * 1e3:.1f} ms; GB/s counted with the same "
                   f"{BYTES_PER_PARAM[kind]} B/param as the GPU so ratios are params/s ratios"),
        "params_per_s": round(n / per, 1),
    }


def cpu_pipeline_baseline(n_batches: int = 24, strategy: str = "optimizer_prediction", depth: int = 4):
    """The reference's executor on config 1 (oracle/runtime_ref.py: the numpy
    float64 restatement of pipesim's 1F1B executor and dense stages, BLAS on
    every host core) over a bounded sample of n_batches synthetic mini-batches:
    samples/s, the first clause of BASELINE.json's metric, on the host."""
    import numpy as np

    from oracle import optim_ref, runtime_ref

    dims, acts, batch = [3072, 1024, 1024, 1024, 10], ["relu", "relu", "relu", "linear"], 128
    rng = np.random.default_rng(0)
    xs = [rng.normal(0, 1, (batch, dims[0])) for _ in range(4)]
    ys = [np.eye(dims[-1])[rng.integers(0, dims[-1], batch)] for _ in range(4)]

    def init(i, din, dout):
        r = np.random.default_rng(100 + i)
        return r.normal(0, (2.0 / din) ** 0.5, (din, dout)), np.zeros((1, dout))

    t0 = time.perf_counter()
    runtime_ref.run(dims, acts, depth, n_batches, strategy, optim_ref.Hyper("adam"),
                    lambda mb: (xs[(mb - 1) % 4], ys[(mb - 1) % 4]), "softmax_xent", lambda mb: 1e-4, init)
    sec = time.perf_counter() - t0
    return {"value": round(n_batches * batch / sec, 1), "unit": "samples/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": (f"oracle/runtime_ref.py (numpy float64 restatement of pipesim's executor) config 1 "
                       f"MLP {dims}, B={batch}, Adam, 1F1B D={depth}, {strategy}, {n_batches} mini-batches "
                       f"(warm-up and drain included) in {sec:.2f} s; numpy BLAS threads = all host cores, "
                       f"optimizer elementwise single-threaded as in the reference")}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_numpy_optimizer(kind: str, logs=(20, 22, 24, 26)):
    """The reference's own call sequence restated in numpy float64
    (oracle/optim_ref.py <- pipesim optim.py:63-155): OptimizerState.step,
    then prediction_direction + predict_weights for the next forward, on one
    (N,) parameter, N = 2^20 .. 2^26. numpy's elementwise
    ufuncs are single-threaded, as in the reference. Best of 2 after a warm-up."""
    import numpy as np

    from oracle import optim_ref

    rows = []
    for lg in logs:
        n = 1 << lg
        rng = np.random.default_rng(lg)
        w = rng.normal(0, 0.02, n)
        opt = optim_ref.OracleOptimizer(optim_ref.Hyper(kind), ["w"])

        def call(w):
            (nw,), _ = opt.step([w], [rng.normal(0, 1e-2, n)], 1e-3)
            (wh,) = optim_ref.predict_weights([nw], 1e-3, 3, opt.prediction_direction([nw]))
            return nw, wh

        w, _ = call(w)
        best = float("inf")
        for _ in range(2):
            g_t = time.perf_counter()
            rng.normal(0, 1e-2, n)  # the gradient draw, subtracted below
            gen = time.perf_counter() - g_t
            t0 = time.perf_counter()
            w, _ = call(w)
            best = min(best, time.perf_counter() - t0 - gen)
        rows.append({"n": n, "ms": round(best * 1e3, 2), "ns_per_param": round(best / n * 1e9, 2),
                     "gbs_equiv": round(BYTES_PER_PARAM[kind] * n / best / 1e9, 3)})
        del w, opt
    return {"cpu": cpu_model(), "threads": 1, "kind": kind,
            "path": "oracle/optim_ref.py OracleOptimizer.step + prediction_direction + predict_weights "
                    "(numpy float64, the reference's evaluation order)", "sizes": rows}


def reference_arm(args):
    """--impl reference: the reference's algorithm for this path on the host
    cores (the oracle's C port, float64 like the reference, OpenMP on every
    core): W warm-up steps then K timed steps, each one K3 pass over a bounded
    2^26-parameter sample. Rank 0 only under torchrun."""
    import numpy as np

    from oracle import c_oracle

    rank, world, _ = dist_env()
    if rank != 0:
        return
    c_oracle.build()
    n = 1 << 26
    rng = np.random.default_rng(0)
    w, g, m = rng.normal(0, 0.02, n), rng.normal(0, 1e-2, n), rng.normal(0, 1e-3, n)
    v = rng.normal(0, 1e-2, n) ** 2 if args.kind != "sgdm" else None
    wh = np.empty(n)
    hp = c_oracle.hp(args.kind)
    t = 10
    for _ in range(max(args.warmup, 1)):
        c_oracle.step_predict(hp, w, g, m, v, wh, 1e-3, 3e-3, t)
        t += 1
    t0 = time.perf_counter()
    for _ in range(args.steps):
        c_oracle.step_predict(hp, w, g, m, v, wh, 1e-3, 3e-3, t)
        t += 1
    per = (time.perf_counter() - t0) / args.steps
    value = round(BYTES_PER_PARAM[args.kind] * n / per / 1e9, 2)
    sample = (f"oracle/c/optim_oracle.c K3 ({args.kind}, float64 like the reference, OpenMP) over {n} params per "
              f"step, {args.steps} timed steps after {max(args.warmup, 1)} warm-up, {per * 1e3:.1f} ms/step; GB/s "
              f"counted with the same {BYTES_PER_PARAM[args.kind]} B/param as the GPU so ratios are params/s ratios")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(per * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"K3 step+predict {args.kind} on the host cores, 2^26-param sample per step "
                               f"(reference algorithm, oracle port; the reference is pure Python)"},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": c_oracle.threads(), "kind": "port",
                         "sample": sample, "params_per_s": round(n / per, 1)},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "vs_baseline": None,
    }
    line["cpu_baseline"]["cpu"] = cpu_model()
    try:
        line["numpy_reference_path"] = cpu_numpy_optimizer(args.kind)
    except Exception as exc:
        line["numpy_reference_path"] = {"error": f"{type(exc).__name__}: {exc}"}
    try:
        line["pipeline"] = {
            "pred_on": cpu_pipeline_baseline(strategy="optimizer_prediction"),
            "pred_off": cpu_pipeline_baseline(strategy="async_raw"),
        }
        line["pipeline"]["value"] = line["pipeline"]["pred_on"]["value"]
        line["pipeline"]["unit"] = "samples/s"
    except Exception as exc:  # the kernel line above must still print
        line["pipeline"] = {"error": f"{type(exc).__name__}: {exc}"}
    print(json.dumps(line), flush=True)


# ---- our arm --------------------------------------------------------------------------------


def kernel_leg(args, torch, dist, rank, world, device):
    from paper_2312_00839_b200 import _lib
    from paper_2312_00839_b200.optim import OptimizerConfig

    lib = _lib.load()
    n = int(args.n_params)
    kind = args.kind
    gen = torch.Generator(device=device)
    mk = lambda seed, scale: torch.randn(n, device=device, generator=gen.manual_seed(seed)) * scale  # noqa: E731
    w = mk(0, 0.02)
    g = mk(1, 1e-2)
    m = mk(2, 1e-3)
    v = mk(3, 1e-2).square_() if kind != "sgdm" else None
    w_hat = torch.empty(n, device=device)
    hp = OptimizerConfig(kind).hparams()
    stream = torch.cuda.current_stream(device)
    lr, s = 1e-3, 3
    t = [10]

    def launch():
        rc = lib.po_step_predict(ctypes.byref(hp), w.data_ptr(), g.data_ptr(), m.data_ptr(),
                                 None if v is None else v.data_ptr(), w_hat.data_ptr(), n, lr, lr * s, t[0], None,
                                 None, stream.cuda_stream)
        _lib.check(rc, "po_step_predict")
        t[0] += 1

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(device.index if device.index is not None else 0)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(device)
    e0.record(stream)
    for _ in range(args.steps):
        launch()
    e1.record(stream)
    torch.cuda.synchronize(device)
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    ms_max = ms
    if world > 1:
        tt = torch.tensor([ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max = float(tt.item())
    bytes_step = BYTES_PER_PARAM[kind] * n
    # every kernel x kind at the same N (BASELINE configs[4] at 1B), same
    # timing regime (back-to-back launches, inputs >> L2), median of 5
    if v is None:
        v = mk(3, 1e-2).square_()
    kinds = {}
    for kd in ("sgdm", "adam", "adamw"):
        hpk = OptimizerConfig(kd).hparams()
        vp = None if kd == "sgdm" else v.data_ptr()
        for kern_name, bpp in (("predict", 12 if kd == "sgdm" else 16), ("step", 20 if kd == "sgdm" else 28),
                               ("step_predict", BYTES_PER_PARAM[kd])):
            def one():
                if kern_name == "predict":
                    rc = lib.po_predict(ctypes.byref(hpk), w.data_ptr(), m.data_ptr(), vp, w_hat.data_ptr(), n,
                                        lr * s, 10, None, stream.cuda_stream)
                elif kern_name == "step":
                    rc = lib.po_step(ctypes.byref(hpk), w.data_ptr(), g.data_ptr(), m.data_ptr(), vp, None, n, lr,
                                     10, None, None, stream.cuda_stream)
                else:
                    rc = lib.po_step_predict(ctypes.byref(hpk), w.data_ptr(), g.data_ptr(), m.data_ptr(), vp,
                                             w_hat.data_ptr(), n, lr, lr * s, 10, None, None, stream.cuda_stream)
                _lib.check(rc, kern_name)

            one()
            ts = []
            for _ in range(3):  # 3 samples of 4 back-to-back launches, median
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                for _ in range(4):
                    one()
                a1.record(stream)
                a1.synchronize()
                ts.append(a0.elapsed_time(a1) / 4)
            t_ms = statistics.median(ts)
            kinds[f"{kern_name}/{kd}"] = {"ms": round(t_ms, 4), "gbs": round(bpp * n / (t_ms * 1e-3) / 1e9, 1)}
    del w, g, m, v, w_hat
    torch.cuda.empty_cache()
    return {"kernels": kinds, "ms_per_step": ms_max, "ms_local": ms, "gbs_per_rank": bytes_step / (ms * 1e-3) / 1e9,
            "value": world * bytes_step / (ms_max * 1e-3) / 1e9, "launches": args.steps, "clocks": clk, "n": n}


def e2e_leg(args, torch, dist, world, device):
    """Same metric through the host-buffer API: pinned host W, G in; W', W_hat out."""
    from paper_2312_00839_b200.optim import HostStreamer, OptimizerConfig, OptimizerState, predict_weights

    n = int(args.n_params)
    if world > 2:
        # 16 B/param of pinned host memory per rank: cap the sample at 2.5e8
        # params (4 GB per rank) so 8 ranks do not pin 128 GB of host RAM —
        # the metric is a rate, and 2.5e8 is still ~15 streamer chunks
        n = min(n, 250_000_000)
    kind = args.kind
    pin = lambda: torch.empty(n, dtype=torch.float32).pin_memory()  # noqa: E731
    w_h, g_h, wo_h, wh_h = pin(), pin(), pin(), pin()
    w_h.normal_(0, 0.02)
    g_h.normal_(0, 1e-2)
    opt = OptimizerState(OptimizerConfig(kind), ["stage.flat"], device=device, eager_checks=False)
    streamer = HostStreamer(device)
    launches = [0]

    def step():
        launches[0] += streamer.step_predict(opt, w_h, g_h, 1e-3, 1e-3, 3, wo_h, wh_h)

    for _ in range(max(1, min(args.warmup, 2))):
        step()
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    launches[0] = 0
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        step()
    e1.record()
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1) / args.e2e_steps
    if world > 1:
        tt = torch.tensor([ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    opt.check_finite()
    # device-resident weights/state, gradient from pinned host memory, the
    # non-finite flag read back (the training-loop setting)
    wd = torch.empty(n, device=device).normal_(0, 0.02)
    whd = torch.empty(n, device=device)
    opt2 = OptimizerState(OptimizerConfig(kind), ["stage.flat"], device=device, eager_checks=False)
    streamer.step_predict_resident(opt2, wd, g_h, 1e-3, 1e-3, 3, whd)
    torch.cuda.synchronize(device)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record()
    res_launches = 0
    for _ in range(args.e2e_steps):
        res_launches += streamer.step_predict_resident(opt2, wd, g_h, 1e-3, 1e-3, 3, whd)
        bad = int(opt2._bad.item())  # the step's result read back every step
        assert bad == (1 << 63) - 1
    r1.record()
    torch.cuda.synchronize(device)
    ms_res = r0.elapsed_time(r1) / args.e2e_steps
    if world > 1:
        tt = torch.tensor([ms_res], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_res = float(tt.item())
    del wd, whd, opt2
    # the reference's own call sequence on host lists (pipesim swaps in
    # OptimizerState.step, then prediction_direction + predict_weights for the
    # next forward: optim.py:63-155): W, G in -> W', dirs out; dirs out; W', d
    # in -> W_hat out — 32 B/param over PCIe, each call chunked and overlapped
    lopt = OptimizerState(OptimizerConfig(kind), ["stage.flat"], device=device, eager_checks=False)

    def list_step():
        new, _ = lopt.step([w_h], [g_h], 1e-3)
        d = lopt.prediction_direction(new)
        return predict_weights(new, 1e-3, 3, d)

    # warm-up calls: the outputs are new pinned host tensors; the first call
    # pins them afresh (~0.4 s per GB), later calls get the outputs the caller
    # dropped back from torch's pinned-host cache (scripts/list_api_probe.py,
    # profiles/r2_list_api_probe.jsonl)
    for _ in range(2):
        list_step()
    torch.cuda.synchronize(device)
    l_steps = max(1, min(3, args.e2e_steps))
    t_l = time.perf_counter()
    for _ in range(l_steps):
        list_step()
    torch.cuda.synchronize(device)
    ms_list = (time.perf_counter() - t_l) / l_steps * 1e3
    del lopt
    # the e2e step's own bound, measured: the same 8 B/param in and 8 B/param
    # out as two plain copies per direction on two streams at once (pinned
    # host <-> device, no kernel)
    d_a, d_b = torch.empty(n, device=device), torch.empty(n, device=device)
    s_in, s_out = torch.cuda.Stream(device), torch.cuda.Stream(device)
    torch.cuda.synchronize(device)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for st_ in (s_in, s_out):
        st_.wait_stream(torch.cuda.current_stream(device))
    with torch.cuda.stream(s_in):
        d_a.copy_(w_h, non_blocking=True)
        d_b.copy_(g_h, non_blocking=True)
    with torch.cuda.stream(s_out):
        wo_h.copy_(d_b, non_blocking=True)
        wh_h.copy_(d_a, non_blocking=True)
    for st_ in (s_in, s_out):
        torch.cuda.current_stream(device).wait_stream(st_)
    p1.record()
    torch.cuda.synchronize(device)
    ms_pcie = p0.elapsed_time(p1)
    del d_a, d_b
    # `e2e` is the reference-shaped round trip: the caller's W and G come from
    # pinned host memory every step and W' and W_hat go back (one fused K3
    # call, HostStreamer.step_predict); the training-loop setting with W, m, v
    # device-resident (only the gradient in, the non-finite flag out) and the
    # three-call list API are reported beside it.
    res = {
        "value": round(world * BYTES_PER_PARAM[kind] * n / (ms * 1e-3) / 1e9, 2),
        "unit": "GB/s",
        "h2d_bytes_per_step": 8 * n,
        "d2h_bytes_per_step": 8 * n,
        "ms_per_step": round(ms, 3),
        "n_params": n,
        "wall_s": round(wall, 3),
        "path": "OptimizerState + HostStreamer.step_predict: pinned host W, G -> device (chunked) -> K3 against "
                "device-resident m, v -> W', W_hat -> pinned host (H2D and D2H streams overlapped)",
        "launches": launches[0],
        "pcie_bound": {
            "ms_per_step": round(ms_pcie, 3),
            "frac": round(ms_pcie / ms, 4),
            "how": "the step's bytes (8 B/param H2D + 8 B/param D2H) as plain pinned copies, both directions at "
                   "once, no kernel: frac = that time / the e2e step time",
        },
        "grad_in_state_resident": {
            "value": round(world * BYTES_PER_PARAM[kind] * n / (ms_res * 1e-3) / 1e9, 2),
            "unit": "GB/s",
            "h2d_bytes_per_step": 4 * n,
            "d2h_bytes_per_step": 8,
            "ms_per_step": round(ms_res, 3),
            "path": "OptimizerState + HostStreamer.step_predict_resident: pinned host G -> device in 16M-element "
                    "chunks (H2D stream) -> K3 per chunk on device-resident W, m, v -> W', W_hat on device; "
                    "non-finite flag read back each step",
            "launches": res_launches,
        },
        "list_api": {
            "value": round(world * BYTES_PER_PARAM[kind] * n / (ms_list * 1e-3) / 1e9, 2),
            "unit": "GB/s",
            "h2d_bytes_per_step": 16 * n,
            "d2h_bytes_per_step": 16 * n,
            "ms_per_step": round(ms_list, 3),
            "steps": l_steps,
            "path": "reference call sequence on host lists: OptimizerState.step([W],[G]) -> (W', dirs); "
                    "prediction_direction(W'); predict_weights(W', lr, 3, d) -> W_hat (each chunked through "
                    "HostStreamer; wall clock)",
        },
    }
    del w_h, g_h, wo_h, wh_h, streamer, opt
    torch.cuda.empty_cache()
    if hasattr(torch._C, "_host_emptyCache"):  # hand the 16 GB of pinned host buffers back to the OS
        torch._C._host_emptyCache()
    return res


def pipeline_leg(args, torch, dist, rank, world, device):
    """Config 1 through the 1F1B runner (+ configs 2-4 unless --no-configs):
    samples/s with prediction on vs off."""
    from paper_2312_00839_b200 import bench_pipeline as bp

    t_leg = time.perf_counter()

    def progress(what):
        print(f"[bench] pipeline leg: {what} done at {time.perf_counter() - t_leg:.1f} s", file=sys.stderr,
              flush=True)

    if world == 1:
        out = bp.single_gpu_pipeline(torch, device, n_batches=args.pipeline_batches)
        progress("config 1 fp32")
        t = bp.single_gpu_pipeline(torch, device, n_batches=args.pipeline_batches, tf32=True, with_eager=False,
                                   with_roofline=False)
        out["tf32"] = {k: t[k] for k in ("pred_on", "pred_off", "prediction_overhead", "serial_streams", "config")}
        progress("config 1 tf32")
        out["projected_8gpu"] = bp.projected_multi_gpu(torch, device, depth=8, n_batches=args.pipeline_batches)
        from paper_2312_00839_b200 import stages as _stages

        _stages.TC_FP32 = False  # the same projection with cuBLAS's SIMT fp32 GEMMs, for reference
        try:
            simt = bp.projected_multi_gpu(torch, device, depth=8, n_batches=args.pipeline_batches)
        finally:
            _stages.TC_FP32 = True
        out["projected_8gpu"]["simt_fp32_gemms"] = {
            "prediction_overhead": simt["prediction_overhead"],
            "pred_off_samples_per_s": simt["pred_off"]["projection"]["one_stage_per_gpu_samples_per_s"],
            "pred_on_samples_per_s": simt["pred_on"]["projection"]["one_stage_per_gpu_samples_per_s"]}
        progress("projected 8-GPU")
        out["depth_sweep_1gpu"] = bp.depth_sweep(torch, device, n_batches=args.pipeline_batches)
        progress("depth sweep")
        try:
            out["strategies"] = bp.strategy_comparison(torch, device, n_batches=args.pipeline_batches)
        except Exception as exc:
            out["strategies"] = {"error": f"{type(exc).__name__}: {exc}"}
        progress("weight-policy comparison")
        out["gpipe"] = {}
        for name, nb in (("config1", args.pipeline_batches), ("config2_vgg16", 32), ("config3_resnet101", 16)):
            try:
                out["gpipe"][name] = bp.gpipe_comparison(torch, device, name, n_batches=nb)
            except Exception as exc:
                out["gpipe"][name] = {"error": f"{type(exc).__name__}: {exc}"}
            progress(f"gpipe vs pipeoptim {name}")
        if not args.no_cpu:
            try:
                out["cpu_baseline"] = cpu_pipeline_baseline()
            except Exception as exc:
                out["cpu_baseline"] = {"error": f"{type(exc).__name__}: {exc}"}
            progress("cpu baseline")
    else:
        staged = args.dist_backend != "nccl"
        out = bp.multi_gpu_pipeline(torch, dist, rank, world, device, n_batches=args.pipeline_batches,
                                    host_staging=staged)
        if world >= 2 and world % 2 == 0:
            from paper_2312_00839_b200.pipeline import bench_hybrid_dp_pp

            try:
                out["hybrid_dp_pp"] = bench_hybrid_dp_pp(torch, dist, rank, world, device, host_staging=staged)
            except Exception as exc:
                out["hybrid_dp_pp"] = {"error": f"{type(exc).__name__}: {exc}"}
    if not args.no_configs:
        from paper_2312_00839_b200.pipeline import bench_module_pipeline

        configs = {}
        for name in bp.MODULE_CONFIGS:
            try:
                if world == 1:
                    # n >= 8 D mini-batches per measured run, fill and drain included
                    n_mb = 8 * bp.MODULE_CONFIGS[name]["depth"]
                    configs[name] = bp.single_gpu_module_pipeline(torch, device, name, n_batches=n_mb)
                    if bp.MODULE_CONFIGS[name].get("channels_last"):  # conv configs: bf16 stage compute too
                        b = bp.single_gpu_module_pipeline(torch, device, name, n_batches=n_mb, amp="bf16",
                                                          with_eager=False, with_roofline=False)
                        configs[name]["bf16"] = {k: b[k] for k in ("config", "pred_off", "pred_on",
                                                                   "prediction_overhead")}
                        configs[name]["bf16"]["semantics"] = (
                            "throughput only: autocast's bf16 weight copies make conv input gradients use the "
                            "forward (predicted) weights, not the live ones (S9); no parity claim")
                else:
                    configs[name] = bench_module_pipeline(torch, dist, rank, world, device, name, n_batches=16,
                                                          host_staging=args.dist_backend != "nccl")
            except Exception as exc:
                configs[name] = {"error": f"{type(exc).__name__}: {exc}"}
            torch.cuda.empty_cache()
            progress(name)
        out["configs"] = configs
    return out


def ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (there is no CPU fallback for the PipeOptim kernels)")
    device = torch.device("cuda", 0 if args.share_gpu else local)
    torch.cuda.set_device(device)
    if world > 1:
        if args.dist_backend == "nccl":
            # keep NCCL's communicator-init lines (rank counts, NVLS/P2P
            # transports) in stderr so a multi-GPU run can be audited
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")
    kern = kernel_leg(args, torch, dist, rank, world, device)
    e2e = None if args.no_e2e else e2e_leg(args, torch, dist, world, device)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.kind)
    line = _line(args, kern, e2e, cpu, world)
    pipe = None
    if not args.no_pipeline:
        # the pipeline leg runs last under a watchdog: a hung NCCL exchange must
        # not cost the kernel measurement — rank 0 then prints the line with the
        # pipeline marked as timed out and every rank exits
        import threading

        def _expire():
            if rank == 0:
                line["pipeline"] = {"error": f"timeout after {args.pipeline_timeout} s"}
                print(json.dumps(line), flush=True)
            os._exit(0)

        import faulthandler

        if args.pipeline_timeout is None:
            args.pipeline_timeout = 420.0 if world == 1 else 900.0

        faulthandler.dump_traceback_later(max(1.0, args.pipeline_timeout - 2.0), exit=False)  # where it hung
        dog = threading.Timer(args.pipeline_timeout, _expire)
        dog.daemon = True
        dog.start()
        try:
            pipe = pipeline_leg(args, torch, dist, rank, world, device)
        except Exception as exc:  # reported, never silently dropped
            pipe = {"error": f"{type(exc).__name__}: {exc}"}
        dog.cancel()
        faulthandler.cancel_dump_traceback_later()
    line["pipeline"] = pipe
    if rank == 0:  # printed before any teardown that could fail
        print(json.dumps(line), flush=True)
    if world > 1:
        try:
            dist.barrier()
            dist.destroy_process_group()
        except Exception:
            os._exit(0)


def _line(args, kern, e2e, cpu, world):
    peak, peak_src = measured_peak()
    traffic = ncu_traffic()
    gbs = kern["gbs_per_rank"]
    launches = kern["launches"]  # our kernels inside the timed region of `value` (one K3 per step)
    line = {
        "metric": METRIC,
        "value": round(kern["value"], 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(kern["ms_per_step"], 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (torch.Generator N(0,.02) W, N(0,1e-2) G, N(0,1e-3) m, N(0,1e-2)^2 v)",
        "config": {
            "workload": f"K3 fused {args.kind} step + weight prediction (s=3) over {kern['n']} fp32 params per GPU "
                        f"(BASELINE configs[4] at 1B; one stage per GPU, replicas only)",
            "n_params_per_gpu": kern["n"],
            "bytes_per_param": BYTES_PER_PARAM[args.kind],
            "l2": "inputs (16 GB) >> 126 MB L2; no flush needed",
            "parallelism": f"replicas{world}",
        },
        "roofline": {
            "bound": "hbm",
            "achieved": round(gbs, 1),
            "peak": peak,
            "unit": "GB/s",
            "frac": round(gbs / peak, 4),
            "frac_of_8tbs": round(gbs / 8000.0, 4),
            "peak_source": peak_src,
            "traffic": (round(traffic["dram_bytes_per_launch"] * kern["n"] / traffic["n"]) if traffic else None),
            "traffic_note": (f"ncu dram__bytes_read+write per launch at n={traffic.get('n')}" if traffic else
                             "no ncu capture committed"),
            "kernel": "po_stream_kernel<ADAM, STEP_PREDICT> (K3)",
            "kernel_ms": round(kern["ms_per_step"], 4),
        },
        "kernels_1e9": kern.get("kernels"),
        "clocks": kern["clocks"],
        "e2e": e2e,
        "gpu_launches": launches,
        "pipeline": None,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    return line


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
