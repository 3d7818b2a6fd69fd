"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
itself (arXiv 2312.00839's pipesim, /root/reference/pkg/src, read-only).

Run in the build container (the reference does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed; small):
  optim_golden.npz     OptimizerState trajectories for sgdm/adam/adamw on fp32-
                       representable inputs: W, state, prediction_direction and
                       predict_weights(s in 1,3,7) after every step.
  schedule_golden.json build_1f1b stage_events / slots / update_gaps / horizon /
                       bubble ratios / makespan for D=1..8, several n.
  runtime_golden.json  execute() reports (losses, VersionRecords, peaks,
                       final versions, final params) for small MLP runs, and
                       the config-1 run (4-stage 3072-1024^3-10 MLP, Adam
                       lr 1e-4, 40 mini-batches) prediction on and off.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from pipesim import experiments as X  # noqa: E402
from pipesim.config import config_from_dict  # noqa: E402
from pipesim.linalg import Matrix, RngStream  # noqa: E402
from pipesim.optim import OptimizerConfig, OptimizerState, predict_weights  # noqa: E402
from pipesim.runtime import BatchSource, build_timeline, execute, update_gaps  # noqa: E402
from pipesim.schedule import bubble_ratio, build_1f1b, makespan, steady_state_window  # noqa: E402
from pipesim.stages import build_layers, build_stages  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def make_optim():
    out = {}
    rng = np.random.default_rng(20231201)
    n, steps = 257, 8
    for kind, extra in (("sgdm", {}), ("sgdm_wd_damp", {"weight_decay": 0.05, "dampening": 0.3}),
                        ("adam", {}), ("adamw", {"decoupled_decay": 0.1})):
        base = kind.split("_")[0]
        cfg = OptimizerConfig(base, **extra)
        w0 = f32(rng.normal(0, 0.02, (1, n)))
        gs = [f32(rng.normal(0, 1e-2, (1, n))) for _ in range(steps)]
        lrs = [1e-3 * (1 + 0.1 * i) for i in range(steps)]
        st = OptimizerState(cfg, ["w"])
        params = [Matrix(w0)]
        out[f"{kind}/w0"] = w0
        out[f"{kind}/grads"] = np.stack(gs)
        out[f"{kind}/lrs"] = np.array(lrs)
        ws, s1, s2, dirs, preds = [], [], [], [], []
        for i, g in enumerate(gs):
            params, _ = st.step(params, [Matrix(g)], lrs[i])
            ws.append(params[0].a.copy())
            if base == "sgdm":
                s1.append(st.momentum_buf[0].a.copy())
                s2.append(np.zeros((1, n)))
            else:
                s1.append(st.exp_avg[0].a.copy())
                s2.append(st.exp_avg_sq[0].a.copy())
            d = st.prediction_direction(params)
            dirs.append(d[0].a.copy())
            preds.append(np.stack([predict_weights(params, 2e-3, s, d)[0].a for s in (1, 3, 7)]))
        out[f"{kind}/w"] = np.stack(ws)
        out[f"{kind}/s1"] = np.stack(s1)
        out[f"{kind}/s2"] = np.stack(s2)
        out[f"{kind}/dir"] = np.stack(dirs)
        out[f"{kind}/pred"] = np.stack(preds)
        out[f"{kind}/hyper"] = np.array(
            [cfg.momentum, cfg.dampening, cfg.weight_decay, cfg.beta1, cfg.beta2, cfg.eps, cfg.decoupled_decay]
        )
    np.savez_compressed(HERE / "optim_golden.npz", **out)


def make_schedule():
    out = []
    for depth in range(1, 9):
        for n in (1, 2, 3, 8, 13):
            tl = build_1f1b(depth, n)
            stages = []
            for k in range(depth):
                evs = tl.stage_events(k)
                stages.append(
                    {
                        "seq": [f"{e.kind[0].upper()}{e.mb}" for e in evs],
                        "slots": [e.slot for e in evs],
                    }
                )
            gaps = update_gaps(tl)
            steady = steady_state_window(tl)
            out.append(
                {
                    "depth": depth,
                    "n": n,
                    "stages": stages,
                    "global": [[e.slot, e.stage, e.kind[0].upper(), e.mb] for e in tl.events],
                    "gaps": [[mb, k, s] for (mb, k), s in sorted(gaps.items())],
                    "horizon": tl.horizon,
                    "bubble": str(bubble_ratio(tl)),
                    "steady": list(steady) if steady else None,
                    "bubble_steady": str(bubble_ratio(tl, *steady)) if steady else None,
                    "makespan": makespan(tl),
                }
            )
    (HERE / "schedule_golden.json").write_text(json.dumps(out, separators=(",", ":")) + "\n")


class RegressionSource(BatchSource):
    """Seeded N(0,1) batches, as pkg/tests/test_runtime.py:22-31."""

    def __init__(self, seed, rows, din, dout):
        self.seed, self.rows, self.din, self.dout = seed, rows, din, dout

    def batch(self, mb):
        r = RngStream(self.seed, f"batch-{mb}")
        return r.normal(self.rows, self.din), r.normal(self.rows, self.dout)


def _report(rep, stages, with_params=True):
    d = {
        "losses": rep.losses,
        "records": [
            [r.mb, r.micro, r.stage, r.forward_version, r.predicted, r.prediction_target,
             r.backward_version, r.live_backward_version]
            for r in rep.records
        ],
        "snapshot_peaks": rep.snapshot_peaks,
        "stash_peaks": rep.stash_peaks,
        "final_versions": rep.final_versions,
        "bubble_overall": rep.bubble_overall,
        "makespan_unit": rep.makespan_unit,
    }
    if with_params:
        d["params"] = [[p.a.tolist() for p in s.params] for s in stages]
    else:
        d["param_sums"] = [[float(np.sum(p.a)) for p in s.params] for s in stages]
        d["param_absmax"] = [[float(np.max(np.abs(p.a))) for p in s.params] for s in stages]
    return d


SMALL_DIMS = [4, 6, 6, 5, 3]
SMALL_ACTS = ["tanh", "tanh", "tanh", "linear"]
DEEP_DIMS = [4, 6, 6, 6, 6, 6, 6, 5, 3]
DEEP_ACTS = ["tanh"] * 7 + ["linear"]


def make_runtime():
    runs = []
    for dims, acts, depths in ((SMALL_DIMS, SMALL_ACTS, (1, 2, 4)), (DEEP_DIMS, DEEP_ACTS, (8,))):
        for depth in depths:
            for strategy in ("async_raw", "optimizer_prediction"):
                for kind, lr in (("sgdm", 0.05), ("adam", 0.01), ("adamw", 0.01)):
                    n = 2 * depth + 10
                    layers = build_layers(dims, acts)
                    stages = build_stages(layers, depth, RngStream(5).substream("params"))
                    cfg = OptimizerConfig(kind, weight_decay=0.0) if kind == "sgdm" else OptimizerConfig(kind)
                    opts = [OptimizerState(cfg, s.param_names) for s in stages]
                    tl = build_timeline(strategy, depth, n)
                    rep = execute(tl, stages, opts, strategy, RegressionSource(101, 8, dims[0], dims[-1]),
                                  "mse", lambda mb, lr=lr: lr)
                    runs.append(
                        {"name": "small", "dims": dims, "acts": acts, "depth": depth, "n": n,
                         "strategy": strategy, "kind": kind, "lr": lr, "init_seed": 5, "data_seed": 101,
                         "rows": 8, "weight_decay": cfg.weight_decay, **_report(rep, stages)}
                    )
    # §8(f) next: the paper's comparison policies and the synchronous schedules
    for strategy, depth, micros in (("weight_stashing", 4, 1), ("two_buffered", 4, 1), ("gpipe", 4, 4),
                                    ("gpipe", 2, 1), ("naive", 4, 1), ("serial", 1, 1), ("spectrain", 4, 1)):
        for kind, lr in (("sgdm", 0.05), ("adam", 0.01)):
            if strategy == "spectrain" and kind != "sgdm":
                continue
            n = 14
            layers = build_layers(SMALL_DIMS, SMALL_ACTS)
            stages = build_stages(layers, depth, RngStream(5).substream("params"))
            cfg = OptimizerConfig(kind, weight_decay=0.0) if kind == "sgdm" else OptimizerConfig(kind)
            opts = [OptimizerState(cfg, s.param_names) for s in stages]
            tl = build_timeline(strategy, depth, n, micros)
            rep = execute(tl, stages, opts, strategy, RegressionSource(101, 8, SMALL_DIMS[0], SMALL_DIMS[-1]),
                          "mse", lambda mb, lr=lr: lr)
            runs.append(
                {"name": "small_extra", "dims": SMALL_DIMS, "acts": SMALL_ACTS, "depth": depth, "n": n,
                 "micros": micros, "strategy": strategy, "kind": kind, "lr": lr, "init_seed": 5, "data_seed": 101,
                 "rows": 8, "weight_decay": cfg.weight_decay, **_report(rep, stages)}
            )
    # config 1: the CPU-reference run, prediction on and off
    for depth in (4,):
        for strategy in ("optimizer_prediction", "async_raw"):
            cfg = config_from_dict(
                {
                    "name": "config1",
                    "seed": 0,
                    "depth": depth,
                    "strategy": strategy,
                    "schedule": {"kind": "1f1b"},
                    "model": {"layer_dims": [3072, 1024, 1024, 1024, 10],
                              "activations": ["relu", "relu", "relu", "linear"]},
                    "optimizer": {"kind": "adam"},
                    "training": {"n_epochs": 2, "batch_size": 128, "lr": 1e-4},
                    "dataset": {"kind": "tiny-classification", "n_samples": 3200, "seed": 1234,
                                "input_dim": 3072, "n_classes": 10, "noise": 32.0},
                }
            )
            res = X.run_experiment(cfg)
            runs.append(
                {"name": "config1", "dims": cfg.model.layer_dims, "acts": cfg.model.activations,
                 "depth": depth, "n": cfg.n_batches, "strategy": strategy, "kind": "adam", "lr": 1e-4,
                 "init_seed": 0, "data_seed": 1234, **_report(res.report, res.stages, with_params=False)}
            )
    (HERE / "runtime_golden.json").write_text(json.dumps(runs, separators=(",", ":")) + "\n")


def make_rng():
    """Philox golden draws (the reference's own, linalg.py:147-167)."""
    out = {
        "root_7_normal": RngStream(7).normal(2, 3).a.tolist(),
        "sub_7_a_b_uniform": RngStream(7).substream("a").substream("b").uniform(1, 4, -1.0, 2.0).a.tolist(),
        "params_0_layer0_head": RngStream(0).substream("params").substream("layer-0").normal(3072, 1024, 3072 ** -0.5).a[0, :8].tolist(),
    }
    (HERE / "rng_golden.json").write_text(json.dumps(out) + "\n")


def make_files():
    """The reference's own report.json / losses.csv / versions.csv for a small
    PipeOptim run (experiments.write_run_outputs, experiments.py:375-392)."""
    import tempfile

    cfg = config_from_dict({
        "name": "files", "seed": 0, "depth": 4, "strategy": "optimizer_prediction",
        "schedule": {"kind": "1f1b"},
        "model": {"layer_dims": [4, 8, 8, 8, 1], "activations": ["tanh", "tanh", "tanh", "linear"]},
        "optimizer": {"kind": "adam"},
        "training": {"n_epochs": 2, "batch_size": 16, "lr": 0.01},
        "dataset": {"kind": "synthetic-regression", "n_samples": 210, "seed": 5, "input_dim": 4,
                    "target_dim": 1, "noise": 0.05},
    })
    res = X.run_experiment(cfg)
    out = HERE / "files"
    out.mkdir(exist_ok=True)
    with tempfile.TemporaryDirectory() as td:
        d = X.write_run_outputs(res, Path(td), "csv")
        for name in ("report.json", "losses.csv", "versions.csv"):
            (out / name).write_text((d / name).read_text())
    (out / "config.json").write_text(json.dumps(cfg.model_dump(mode="json"), indent=2, sort_keys=True) + "\n")


if __name__ == "__main__":
    make_files()
    make_optim()
    make_schedule()
    make_rng()
    make_runtime()
    for p in sorted(HERE.glob("*golden*")):
        print(p.name, p.stat().st_size)
