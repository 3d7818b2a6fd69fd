"""Pipeline legs of bench.py: config 1 (4-stage 3072-1024^3-10 MLP, ReLU x3 +
linear, softmax cross-entropy, B = 128, Adam lr 1e-4) on synthetic
CIFAR-10-shaped batches resident in HBM, 1F1B with prediction on
(optimizer_prediction) vs off (async_raw, the prediction-disabled control).
"""

from __future__ import annotations

import math
import time

CONFIG1_DIMS = [3072, 1024, 1024, 1024, 10]
CONFIG1_ACTS = ["relu", "relu", "relu", "linear"]
BATCH = 128


class DeviceBatches:
    """Synthetic x ~ N(0,1) (B, 3072) and one-hot labels uniform over 10,
    pre-generated on the device (inputs resident in HBM)."""

    def __init__(self, torch, device, n_distinct: int = 16, seed: int = 0, dims=CONFIG1_DIMS):
        g = torch.Generator(device=device).manual_seed(seed)
        self.x = [torch.randn(BATCH, dims[0], device=device, generator=g) for _ in range(n_distinct)]
        self.y = []
        for _ in range(n_distinct):
            lab = torch.randint(0, dims[-1], (BATCH,), device=device, generator=g)
            self.y.append(torch.nn.functional.one_hot(lab, dims[-1]).float())

    def batch(self, mb: int):
        i = (mb - 1) % len(self.x)
        return self.x[i], self.y[i]


def _run_once(torch, device, strategy, depth, n_batches, data, seed=0, dims=CONFIG1_DIMS, acts=CONFIG1_ACTS):
    from .optim import OptimizerConfig, OptimizerState
    from .runtime import build_timeline, execute
    from .stages import build_layers, build_stages, torch_init

    stages = build_stages(build_layers(dims, acts), depth, torch_init(seed, device), device=device)
    opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=device) for s in stages]
    tl = build_timeline(strategy, depth, n_batches)
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    rep = execute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: 1e-4, checks="deferred")
    e1.record()
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    return rep, e0.elapsed_time(e1) / 1e3, wall


def _graph_for(torch, device, strategy, depth, n_batches, data, seed=0, dims=CONFIG1_DIMS, acts=CONFIG1_ACTS,
               streams="serial"):
    from .optim import OptimizerConfig, OptimizerState
    from .runtime import GraphedExecute, build_timeline
    from .stages import build_layers, build_stages, torch_init

    stages = build_stages(build_layers(dims, acts), depth, torch_init(seed, device), device=device)
    opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=device) for s in stages]
    tl = build_timeline(strategy, depth, n_batches)
    g = GraphedExecute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: 1e-4, warmup_runs=1,
                       streams=streams)
    g.replay()  # first replay: graph upload
    torch.cuda.synchronize(device)
    return g


def _time_replays(torch, device, g, replays):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(replays):
        g.replay()
    e1.record()
    torch.cuda.synchronize(device)
    return e0.elapsed_time(e1) / 1e3 / replays


def _graphed_pair(torch, device, depth, n_batches, data, replays, trials=9, streams=("stage", "serial"),
                  dims=CONFIG1_DIMS, acts=CONFIG1_ACTS):
    """Prediction off/on graphs (per stream mode) timed in alternation (median
    of `trials`), so clock and thermal drift hit every arm alike."""
    import statistics

    graphs = {(s, m): _graph_for(torch, device, s, depth, n_batches, data, streams=m, dims=dims, acts=acts)
              for m in streams for s in ("async_raw", "optimizer_prediction")}
    times = {k: [] for k in graphs}
    for _ in range(trials):
        for k, g in graphs.items():
            times[k].append(_time_replays(torch, device, g, replays))
    return {k: (graphs[k].report(), statistics.median(times[k]), graphs[k].launches, times[k]) for k in graphs}


def _unit_graph(torch, device, k, st, opt, data, loss_kind, predictive, depth, units: int = 1):
    """CUDA graph of stage k's work for `units` consecutive mini-batches:
    forward (+ loss on the last stage) + backward + update (K3 when
    predictive and not last, else K2), back to back as on the stage's own
    GPU in the 1F1B steady state."""
    from .runtime import staging_in_grad_ok

    last = k == depth - 1
    x0, y0 = data.batch(1)
    x = x0 if k == 0 else torch.randn((x0.shape[0], *st.in_shape), device=device)
    g_last = None if last else torch.randn((x0.shape[0], *st.out_shape), device=device)
    predicted = predictive and not last
    # as in the pipeline: W_hat over the dead gradient where that is exact,
    # and the predicted forward reads it (the run's F_{j+D-k} after U_j)
    if predicted and staging_in_grad_ok(st, True, 1):
        staging = st.flat.grad
    else:
        staging = st.flat.layout.empty(device)
        if predicted:
            staging.copy_(st.flat.data)
    fwd_weights = st.flat.layout.views(staging) if predicted else st.params
    opt._bind(st.flat.layout)
    opt._ensure_state()

    from . import stages as _stages
    from .stages import StageModel

    defer = _stages.FUSE_WGRAD_UPDATE and isinstance(st, StageModel)  # as the runners do

    def unit():
        if last:
            g = st.run_forward_loss(fwd_weights, (0, 0), x, 1, y0, loss_kind, check_finite=False)[2]
        else:
            st.run_forward(fwd_weights, (0, 0), x, 1, check_finite=False)
            g = g_last
        if defer:
            st.run_backward(st.params, (0, 0), g, need_input_grad=k > 0, defer_wgrad=True)
            wg = st.take_deferred_wgrad()
        else:
            st.run_backward(st.params, (0, 0), g, need_input_grad=k > 0)
            wg = []
        if predictive and not last:
            if wg:
                opt.step_fused_(st.flat, 1e-4, 1e-4, depth - k - 1, staging, wg)
            else:
                opt.step_predict_(st.flat, 1e-4, 1e-4, depth - k - 1, staging)
        elif wg:
            opt.step_fused_(st.flat, 1e-4, 0.0, 0, None, wg)
        else:
            opt.step_(st.flat, 1e-4)

    opt.eager_checks = False
    for _ in range(2):
        unit()
    torch.cuda.synchronize(device)
    graph = torch.cuda.CUDAGraph()
    from .runtime import capture

    with capture(graph):
        for _ in range(units):
            unit()
    graph.replay()
    torch.cuda.synchronize(device)
    # the graph replays into these addresses: keep the buffers allocated
    # outside the capture alive as long as the graph
    graph.keepalive = (staging, x, g_last, y0)
    return graph


UNITS_PER_GRAPH = 16


def stage_unit_times(torch, device, make, data, loss_kind, reps: int = 5, trials: int = 9,
                     units: int | None = None, shared: bool = True):
    """Per-stage device time of one mini-batch's work — SURVEY.md §8d's
    t_f,k + t_b,k (+ t_u,k) — with prediction off (K2 update) and on (K3),
    each captured as `units` back-to-back units in one CUDA graph (the
    stage's steady state on its own GPU; one unit per graph would add a
    graph launch gap to every unit) on THROWAWAY stages from `make()` ->
    (stages, opts) — one set shared by both modes unless shared=False —
    (replays train them),
    the two modes replayed in alternation (`reps` replays per sample, median
    of `trials`) so that drift hits both alike. Returns {"pred_off": [s per stage], "pred_on": [...]}."""
    units = UNITS_PER_GRAPH if units is None else units
    import statistics

    out = {"pred_off": [], "pred_on": []}
    # shared: both modes on the SAME stage buffers — a separate build places
    # them at other addresses (other L2 slices / pages), which moved a config-1
    # unit by ~0.5 us between builds, as much as the prediction's own cost
    # (profiles/r2_unit_shape_probe.jsonl); replays of either graph only
    # advance the shared weights and state. Module stages (configs 2-4) are
    # measured on separate builds: one ModuleStage under two captured graphs
    # slows both of GNMT-8's stage-0 units by the same 0.085 ms
    # (profiles/r2_unit_times_shared_buffers.jsonl)
    if shared:
        one = make()
        sets = {key: one for key in out}
    else:
        sets = {key: make() for key in out}
    depth = len(sets["pred_off"][0])
    for k in range(depth):
        graphs = {key: _unit_graph(torch, device, k, sets[key][0][k], sets[key][1][k], data, loss_kind,
                                   key == "pred_on", depth, units) for key in out}
        samples = {key: [] for key in out}
        for _ in range(trials):
            for key, graph in graphs.items():
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    graph.replay()
                e1.record()
                torch.cuda.synchronize(device)
                samples[key].append(e0.elapsed_time(e1) / 1e3 / (reps * units))
        for key in out:
            out[key].append(statistics.median(samples[key]))
        del graphs
    return out


def unit_time_projection(stage_times, batch, n, depth):
    """Throughput PROJECTED from measured per-stage unit times (not a bound):
    one stage per GPU runs at B / max_k t_k * n / (n + D - 1) (1F1B unit
    makespan 2n + 2D - 2); all stages serialised on one stream at B / sum_k t_k."""
    return {"one_stage_per_gpu_samples_per_s": round(batch / max(stage_times) * n / (n + depth - 1), 1),
            "serialised_samples_per_s": round(batch / sum(stage_times), 1),
            "stage_ms": [round(t * 1e3, 4) for t in stage_times]}


def _attach_bounds(row, bound, projection=None):
    """row["roofline"] = the counted-work bounds (roofline.py); the fraction
    is achieved / the single-GPU bound (all stages share this GPU)."""
    row["roofline"] = bound
    row["frac_of_roofline"] = round(row["samples_per_s"] / bound["single_gpu"]["samples_per_s"], 4)
    if projection is not None:
        row["projection"] = projection


def single_gpu_pipeline(torch, device, n_batches: int = 64, depth: int = 4, replays: int = 5, tf32: bool = False,
                        with_eager: bool = True, with_roofline: bool = True):
    """All `depth` stages on one GPU (the single-GPU 1F1B runner). Each
    measured unit is one full run of the 1F1B timeline (n_batches
    mini-batches, warm-up and drain included), replayed from a CUDA graph
    (`GraphedExecute`). Headline: the stage-concurrent runner (one CUDA stream
    per stage, `streams="stage"`); the serialised runner (every event on one
    stream, timeline order) and the eager (Python-driven) runner beside it.
    Samples/s with prediction on and off, and the pipeline roofline from
    per-stage graphed unit times."""
    from .optim import OptimizerConfig, OptimizerState
    from .stages import build_layers, build_stages, torch_init

    torch.backends.cuda.matmul.allow_tf32 = tf32
    data = DeviceBatches(torch, device)
    out = {"config": f"config1 MLP {CONFIG1_DIMS}, B={BATCH}, Adam lr 1e-4, 1F1B D={depth} on 1 GPU "
                     f"(single-process runner, one CUDA stream per stage, CUDA-graph replay of whole "
                     f"{n_batches}-mini-batch runs), {'TF32' if tf32 else 'fp32 (TF32 off)'} GEMMs"
                     f"{'' if tf32 or depth < 4 else ' (4 K slices, 128-wide tiles while the stages share the GPU)'}, "
                     f"fp32 master weights"}
    launches = 0
    pair = _graphed_pair(torch, device, depth, n_batches, data, replays)
    if with_roofline:
        def make():
            st = build_stages(build_layers(CONFIG1_DIMS, CONFIG1_ACTS), depth, torch_init(7, device), device=device)
            return st, [OptimizerState(OptimizerConfig("adam"), s_.param_names, device=device) for s_ in st]

        units = stage_unit_times(torch, device, make, data, "softmax_xent")
        from .roofline import mlp_pipeline_bounds

        arith = "tf32" if tf32 else "fast_fp32"
        probe = make()[0]
        bounds = {key: mlp_pipeline_bounds(probe, BATCH, n_batches, "adam", key == "pred_on", arith)
                  for key in ("pred_off", "pred_on")}
        del probe
    out["serial_streams"] = {}
    for strategy in ("async_raw", "optimizer_prediction"):
        key = "pred_on" if strategy == "optimizer_prediction" else "pred_off"
        for mode in ("stage", "serial"):
            rep, sec, n_launch, trials = pair[(strategy, mode)]
            row = {"samples_per_s": round(n_batches * BATCH / sec, 1), "s_per_run": round(sec, 5),
                   "s_per_run_trials": [round(t, 5) for t in trials],
                   "final_loss": rep.losses[-1], "optimizer_launches_per_run": n_launch}
            if mode == "stage":
                out[key] = row
            else:
                out["serial_streams"][key] = row
            launches += n_launch * replays
        if with_eager:
            _run_once(torch, device, strategy, depth, min(n_batches, 2 * depth + 2), data)  # eager warm-up
            _, esec, _ = _run_once(torch, device, strategy, depth, n_batches, data)
            out[key]["eager_samples_per_s"] = round(n_batches * BATCH / esec, 1)
        if with_roofline:
            _attach_bounds(out[key], bounds[key], unit_time_projection(units[key], BATCH, n_batches, depth))
            ser = out["serial_streams"][key]
            ser["frac_of_roofline"] = round(ser["samples_per_s"] / bounds[key]["single_gpu"]["samples_per_s"], 4)
    on, off = out["pred_on"]["samples_per_s"], out["pred_off"]["samples_per_s"]
    out["value"] = on
    out["unit"] = "samples/s"
    out["prediction_overhead"] = round(1.0 - on / off, 4)
    ser = out["serial_streams"]
    ser["prediction_overhead"] = round(1.0 - ser["pred_on"]["samples_per_s"] / ser["pred_off"]["samples_per_s"], 4)
    if with_roofline:
        # one stage per GPU (the north star's setting): the pipeline runs at the
        # slowest stage's unit time, so the prediction overhead there is the
        # bottleneck stage's K3-vs-K2 cost (each GPU's L2 holds one stage)
        r_on, r_off = out["pred_on"]["projection"], out["pred_off"]["projection"]
        out["projected_one_stage_per_gpu_prediction_overhead"] = round(
            1.0 - r_on["one_stage_per_gpu_samples_per_s"] / r_off["one_stage_per_gpu_samples_per_s"], 4)
        out["single_gpu_note"] = ("all stages share one GPU's SMs and 126 MB L2 here; W_hat lives in each "
                                  "stage's dead gradient buffer (runtime.STAGING_IN_GRAD), so prediction adds "
                                  "no buffer to the ~105 MB per-mini-batch working set")
    if with_eager:
        out["eager_prediction_overhead"] = round(
            1.0 - out["pred_on"]["eager_samples_per_s"] / out["pred_off"]["eager_samples_per_s"], 4)
    out["launches"] = launches
    torch.backends.cuda.matmul.allow_tf32 = False
    return out


def depth_sweep(torch, device, depths=(1, 2, 4, 8), n_batches: int = 64, replays: int = 5, trials: int = 5):
    """Config 1 at D = 1, 2, 4, 8 pipeline stages on the one GPU (the
    stage-concurrent graphed runner; prediction off/on in alternation). D <= 4
    partitions config 1's four layers; D = 8 widens it to eight layers (one
    more 1024-wide ReLU layer per extra stage, as bench.py --gpus 8 does)."""
    torch.backends.cuda.matmul.allow_tf32 = False
    out = {}
    for d in depths:
        dims = CONFIG1_DIMS if d <= 4 else [3072] + [1024] * (d - 1) + [10]
        acts = CONFIG1_ACTS if d <= 4 else ["relu"] * (d - 1) + ["linear"]
        data = DeviceBatches(torch, device, dims=dims)
        pair = _graphed_pair(torch, device, d, n_batches, data, replays, trials=trials, streams=("stage",),
                             dims=dims, acts=acts)
        row = {"dims": dims}
        for strategy, key in (("async_raw", "pred_off"), ("optimizer_prediction", "pred_on")):
            _, sec, _, _ = pair[(strategy, "stage")]
            row[key] = round(n_batches * BATCH / sec, 1)
        row["prediction_overhead"] = round(1.0 - row["pred_on"] / row["pred_off"], 4)
        out[f"D{d}"] = row
        del pair
        torch.cuda.empty_cache()
    return out


def projected_multi_gpu(torch, device, depth: int = 8, n_batches: int = 64, tf32: bool = False):
    """The north-star setting (one stage per GPU, D = 8) projected from
    per-stage graphed unit times measured on this GPU: config 1 widened to
    8 layers (one more 1024-wide ReLU layer per extra stage, as bench.py
    --gpus 8 runs it). Pipeline throughput = the slowest stage's unit time
    with the 1F1B fill/drain factor n/(n+D-1); the NVLink term (0.5 MB
    activation per boundary at 770 GB/s) is ~1000x faster and not binding."""
    from .optim import OptimizerConfig, OptimizerState
    from .stages import build_layers, build_stages, torch_init

    torch.backends.cuda.matmul.allow_tf32 = tf32
    dims = [3072] + [1024] * (depth - 1) + [10]
    acts = ["relu"] * (depth - 1) + ["linear"]
    data = DeviceBatches(torch, device, dims=dims)
    out = {"config": f"MLP {dims}, B={BATCH}, Adam, D={depth} (one stage per GPU), "
                     f"{'TF32' if tf32 else 'fp32'} GEMMs; projected from per-stage graphed unit times"}
    def make():
        st = build_stages(build_layers(dims, acts), depth, torch_init(11, device), device=device)
        return st, [OptimizerState(OptimizerConfig("adam"), s_.param_names, device=device) for s_ in st]

    units = stage_unit_times(torch, device, make, data, "softmax_xent")
    from .roofline import mlp_pipeline_bounds

    probe = make()[0]
    for key in ("pred_off", "pred_on"):
        proj = unit_time_projection(units[key], BATCH, n_batches, depth)
        bound = mlp_pipeline_bounds(probe, BATCH, n_batches, "adam", key == "pred_on", "tf32" if tf32 else "fast_fp32")
        out[key] = {"projection": proj, "roofline": bound["one_stage_per_gpu"], "per_stage": bound["per_stage"],
                    "frac_of_roofline": round(proj["one_stage_per_gpu_samples_per_s"] /
                                              bound["one_stage_per_gpu"]["samples_per_s"], 4)}
    del probe
    out["prediction_overhead"] = round(
        1.0 - out["pred_on"]["projection"]["one_stage_per_gpu_samples_per_s"] /
        out["pred_off"]["projection"]["one_stage_per_gpu_samples_per_s"], 4)
    torch.backends.cuda.matmul.allow_tf32 = False
    return out


MODULE_CONFIGS = {
    # BASELINE configs[1..3] (SURVEY.md §8d pipeline synthetic inputs)
    "config2_vgg16": dict(blocks="vgg16", in_shape=(3, 32, 32), classes=100, batch=128, depth=4, opt="sgdm", lr=0.01,
                          channels_last=True),
    # ResNet-101's stage kernels fill the GPU on their own: serialised stages
    # with cuDNN batch norm beat concurrent stages with the grid-safe one (+5 %)
    "config3_resnet101": dict(blocks="resnet101", in_shape=(3, 224, 224), classes=200, batch=64, depth=8,
                              opt="adamw", lr=1e-3, channels_last=True, single_gpu_streams="serial"),
    "config4_gnmt8": dict(blocks="gnmt8", in_shape=(50,), classes=32000, batch=64, depth=8, opt="adam", lr=1e-3,
                          tokens=True),
}


def make_blocks(name: str, classes: int):
    from .stage_models import gnmt8_blocks, resnet101_blocks, vgg16_cifar_blocks

    return {"vgg16": lambda: vgg16_cifar_blocks(classes), "resnet101": lambda: resnet101_blocks(classes),
            "gnmt8": lambda: gnmt8_blocks(classes, 1024)}[name]()


class ModuleBatches:
    def __init__(self, torch, device, cfg, n_distinct=4, seed=0):
        g = torch.Generator(device=device).manual_seed(seed)
        b, shape, c = cfg["batch"], cfg["in_shape"], cfg["classes"]
        if cfg.get("tokens"):
            self.x = [torch.randint(0, c, (b, *shape), device=device, generator=g).float() for _ in range(n_distinct)]
        else:
            self.x = [torch.randn((b, *shape), device=device, generator=g) for _ in range(n_distinct)]
        self.y = [torch.nn.functional.one_hot(torch.randint(0, c, (b,), device=device, generator=g), c).float()
                  for _ in range(n_distinct)]

    def batch(self, mb):
        i = (mb - 1) % len(self.x)
        return self.x[i], self.y[i]


_COSTS: dict = {}


def module_block_costs(torch, name, device):
    """Profiled per-block costs (cached). Multi-rank callers must use ONE
    rank's costs everywhere: timing noise would otherwise give the ranks
    different partitions and mismatched activation shapes."""
    from .stage_models import profile_block_costs

    cfg = MODULE_CONFIGS[name]
    in_dtype = torch.long if cfg.get("tokens") else torch.float32
    if name not in _COSTS:
        _COSTS[name] = profile_block_costs(make_blocks(cfg["blocks"], cfg["classes"]), cfg["in_shape"], cfg["batch"],
                                           device, in_dtype=in_dtype, channels_last=cfg.get("channels_last", False))
    return _COSTS[name]


def module_stages_for(torch, name, device, depth=None, costs=None, amp=None):
    from .stage_models import build_module_stages

    cfg = MODULE_CONFIGS[name]
    depth = depth or cfg["depth"]
    in_dtype = torch.long if cfg.get("tokens") else torch.float32
    costs = costs if costs is not None else module_block_costs(torch, name, device)
    torch.manual_seed(0)
    blocks = make_blocks(cfg["blocks"], cfg["classes"])
    amp_dtype = {None: None, "bf16": torch.bfloat16}[amp]
    return build_module_stages(blocks, depth, device, cfg["in_shape"], costs=costs, in_dtype=in_dtype,
                               channels_last=cfg.get("channels_last", False), amp_dtype=amp_dtype), costs


def _module_setup(torch, device, name, strategy, n_batches, amp=None):
    """Stages for the single-GPU runs: every stage shares the one GPU, so the
    LSTM recurrences use the SM-time-efficient unsplit GEMMs."""
    from .optim import OptimizerConfig, OptimizerState
    from .runtime import build_timeline
    from .stage_models import set_lstm_split_k

    cfg = MODULE_CONFIGS[name]
    stages, _ = module_stages_for(torch, name, device, amp=amp)
    set_lstm_split_k(stages, False)
    kw = {"weight_decay": 5e-4} if cfg["opt"] == "sgdm" else {}
    opts = [OptimizerState(OptimizerConfig(cfg["opt"], **kw), s.param_names, device=device) for s in stages]
    return stages, opts, build_timeline(strategy, cfg["depth"], n_batches)


def single_gpu_module_pipeline(torch, device, name: str, n_batches: int = 16, tf32: bool = True, trials: int = 3,
                               with_eager: bool = True, with_roofline: bool = True, amp: str | None = None):
    """Configs 2-4 through the single-GPU 1F1B runner (all D stages on one
    GPU). Headline: whole n_batches-mini-batch runs captured into CUDA graphs
    with one stream per stage (`GraphedExecute(streams="stage")`), prediction
    off/on replayed in alternation (median of `trials`); the eager serial
    runner beside it; the pipeline roofline from per-stage graphed unit times
    (SURVEY.md §8d)."""
    import statistics

    from .optim import OptimizerConfig, OptimizerState
    from .runtime import GraphedExecute, execute

    cfg = MODULE_CONFIGS[name]
    torch.backends.cuda.matmul.allow_tf32 = tf32
    torch.backends.cudnn.allow_tf32 = tf32
    data = ModuleBatches(torch, device, cfg)
    lr = cfg["lr"]
    streams = cfg.get("single_gpu_streams", "stage")
    lanes = "one CUDA stream per stage" if streams == "stage" else "stages serialised on one stream, cuDNN batch norm"
    out = {"config": f"{name}: D={cfg['depth']} stages on 1 GPU (single-process runner, {lanes}, "
                     f"CUDA-graph replay of whole {n_batches}-mini-batch runs), batch {cfg['batch']}, "
                     f"{cfg['opt']} lr {lr}, "
                     f"{'bf16 autocast' if amp == 'bf16' else 'TF32' if tf32 else 'fp32'} convs/GEMMs, "
                     f"fp32 master weights",
           "data": f"synthetic, throughput only: {len(data.x)} random batches cycled, so final_loss measures "
                   f"memorisation, not convergence (the reference has no conv/LSTM stages: loss parity is "
                   f"unpinned, SURVEY.md 8(c)); GNMT-8 is an LSTM stack with a last-position vocabulary head, "
                   f"no attention"}
    try:
        graphs = {}
        for strategy in ("async_raw", "optimizer_prediction"):
            stages, opts, tl = _module_setup(torch, device, name, strategy, n_batches, amp)
            if streams == "serial":  # one stream: cuDNN's grid-synchronising batch norm is safe
                from .stage_models import use_cudnn_bn

                use_cudnn_bn(stages)
            graphs[strategy] = (GraphedExecute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: lr,
                                               warmup_runs=1, streams=streams), stages)
            graphs[strategy][0].replay()
            torch.cuda.synchronize(device)
        times = {s: [] for s in graphs}
        for _ in range(trials):
            for s, (g, _) in graphs.items():
                times[s].append(_time_replays(torch, device, g, 1))
        for s, (g, stages) in graphs.items():
            key = "pred_on" if s == "optimizer_prediction" else "pred_off"
            sec = statistics.median(times[s])
            out[key] = {"samples_per_s": round(n_batches * cfg["batch"] / sec, 2), "s_per_run": round(sec, 4),
                        "s_per_run_trials": [round(t, 4) for t in times[s]],
                        "final_loss": g.report().losses[-1], "optimizer_launches_per_run": g.launches}
        out["stage_params"] = [s.numel for s in graphs["async_raw"][1]]
        out["boundary_bytes"] = [4 * cfg["batch"] * math.prod(s.out_shape) for s in graphs["async_raw"][1][:-1]]
    finally:
        graphs = g = stages = opts = None  # noqa: F841 (drop the graphs' memory pools)
        torch.cuda.empty_cache()
    if with_roofline:
        def make():
            # one stage per GPU: its work is alone on the device, so cuDNN's
            # (grid-synchronising, faster) batch norm is safe there
            from .stage_models import use_cudnn_bn

            st, _ = module_stages_for(torch, name, device, amp=amp)
            use_cudnn_bn(st)
            kw = {"weight_decay": 5e-4} if cfg["opt"] == "sgdm" else {}
            return st, [OptimizerState(OptimizerConfig(cfg["opt"], **kw), s.param_names, device=device) for s in st]

        units = stage_unit_times(torch, device, make, data, "softmax_xent", reps=3, trials=3, units=4,
                                 shared=False)
        from .roofline import module_pipeline_bounds

        arith = "bf16" if amp == "bf16" else ("tf32" if tf32 else "fast_fp32")
        probe = make()[0]
        in_dtype = torch.long if cfg.get("tokens") else None
        bounds = {key: module_pipeline_bounds(torch, probe, cfg["batch"], n_batches, cfg["opt"], key == "pred_on",
                                              arith, in_dtype=in_dtype) for key in ("pred_off", "pred_on")}
        del probe
        torch.cuda.empty_cache()
    for strategy in ("async_raw", "optimizer_prediction"):
        key = "pred_on" if strategy == "optimizer_prediction" else "pred_off"
        if with_eager:
            stages, opts, tl = _module_setup(torch, device, name, strategy, n_batches, amp)
            torch.cuda.synchronize(device)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            execute(tl, stages, opts, strategy, data, "softmax_xent", lambda mb: lr, checks="deferred")
            e1.record()
            torch.cuda.synchronize(device)
            out[key]["eager_serial_samples_per_s"] = round(n_batches * cfg["batch"] / (e0.elapsed_time(e1) / 1e3), 2)
            del stages, opts
        if with_roofline:
            _attach_bounds(out[key], bounds[key], unit_time_projection(units[key], cfg["batch"], n_batches,
                                                                       cfg["depth"]))
        torch.cuda.empty_cache()
    on, off = out["pred_on"]["samples_per_s"], out["pred_off"]["samples_per_s"]
    out.update(value=on, unit="samples/s", prediction_overhead=round(1.0 - on / off, 4))
    if with_roofline:
        r_on, r_off = out["pred_on"]["projection"], out["pred_off"]["projection"]
        out["projected_one_stage_per_gpu_prediction_overhead"] = round(
            1.0 - r_on["one_stage_per_gpu_samples_per_s"] / r_off["one_stage_per_gpu_samples_per_s"], 4)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    return out


def multi_gpu_pipeline(torch, dist, rank, world, device, n_batches: int = 64, host_staging: bool = False):
    """One stage per GPU over NCCL (pipeline.py); depth = world."""
    from .pipeline import bench_config1_pipeline

    return bench_config1_pipeline(torch, dist, rank, world, device, n_batches=n_batches, host_staging=host_staging)


def gpipe_comparison(torch, device, name: str = "config1", n_batches: int = 64, micros: int = 4, trials: int = 5,
                     tf32: bool | None = None):
    """The paper's throughput comparison: GPipe (T
    micro-batches per mini-batch, gradients averaged over them before one
    synchronous update per stage; schedule.py:114-147, runtime.py:441-454)
    vs PipeOptim (1F1B with prediction) on the same stages, batch and GPU.
    Both are whole-run CUDA graphs on the stage-concurrent single-GPU runner,
    replayed in alternation (median of `trials`)."""
    import statistics

    from .optim import OptimizerConfig, OptimizerState
    from .runtime import GraphedExecute, build_timeline
    from .stages import build_layers, build_stages, torch_init

    if name == "config1":
        tf32 = False if tf32 is None else tf32
        torch.backends.cuda.matmul.allow_tf32 = tf32
        data, batch, depth, lr, loss = DeviceBatches(torch, device), BATCH, 4, 1e-4, "softmax_xent"

        def setup(strategy):
            st = build_stages(build_layers(CONFIG1_DIMS, CONFIG1_ACTS), depth, torch_init(0, device), device=device)
            return st, [OptimizerState(OptimizerConfig("adam"), s.param_names, device=device) for s in st]
        streams = "stage"
    else:
        cfg = MODULE_CONFIGS[name]
        tf32 = True if tf32 is None else tf32
        torch.backends.cuda.matmul.allow_tf32 = tf32
        torch.backends.cudnn.allow_tf32 = tf32
        data, batch, depth, lr, loss = ModuleBatches(torch, device, cfg), cfg["batch"], cfg["depth"], cfg["lr"], \
            "softmax_xent"

        def setup(strategy):
            st, opts, _ = _module_setup(torch, device, name, strategy, n_batches)
            return st, opts
        streams = cfg.get("single_gpu_streams", "stage")
    graphs = {}
    try:
        for strategy, t in (("gpipe", micros), ("optimizer_prediction", 1)):
            st, opts = setup(strategy)
            if streams == "serial" and name != "config1":
                from .stage_models import use_cudnn_bn

                use_cudnn_bn(st)
            tl = build_timeline(strategy, depth, n_batches, t)
            g = GraphedExecute(tl, st, opts, strategy, data, loss, lambda mb: lr, warmup_runs=1, streams=streams)
            g.replay()
            torch.cuda.synchronize(device)
            graphs[strategy] = g
        times = {s: [] for s in graphs}
        for _ in range(trials):
            for s, g in graphs.items():
                times[s].append(_time_replays(torch, device, g, 1))
        sps = {s: n_batches * batch / statistics.median(v) for s, v in times.items()}
        out = {"config": f"{name}: D={depth}, batch {batch}, {n_batches} mini-batches per run, GPipe T={micros} "
                         f"micro-batches of {batch // micros}; {'TF32' if tf32 else 'fp32'}; one GPU, "
                         f"{'one stream per stage' if streams == 'stage' else 'stages on one stream'}",
               "gpipe_samples_per_s": round(sps["gpipe"], 1),
               "pipeoptim_samples_per_s": round(sps["optimizer_prediction"], 1),
               "pipeoptim_over_gpipe": round(sps["optimizer_prediction"] / sps["gpipe"], 4),
               "gpipe_final_loss": graphs["gpipe"].report().losses[-1],
               "pipeoptim_final_loss": graphs["optimizer_prediction"].report().losses[-1]}
    finally:
        graphs = g = st = opts = None  # noqa: F841
        torch.cuda.empty_cache()
        torch.backends.cuda.matmul.allow_tf32 = False
        torch.backends.cudnn.allow_tf32 = False
    return out


def strategy_comparison(torch, device, n_batches: int = 64, trials: int = 5):
    """SURVEY.md §8(f) rows 1-2 at the same measurement bar as the headline:
    config 1 (fp32, Adam lr 1e-4, D = 4, stage-concurrent whole-run CUDA
    graphs on one GPU, replayed in alternation) under every 1F1B weight
    policy — async_raw (no prediction), PipeDream weight stashing, PipeDream
    2BW, PipeOptim — plus GPipe (T = 4): samples/s, the weight-version memory
    peaks of the reference's report (snapshot_peaks, runtime.py:66-154) and
    the run's final loss."""
    import statistics

    from .optim import OptimizerConfig, OptimizerState
    from .runtime import GraphedExecute, build_timeline
    from .stages import build_layers, build_stages, torch_init

    torch.backends.cuda.matmul.allow_tf32 = False
    data = DeviceBatches(torch, device)
    graphs = {}
    try:
        for strategy, t in (("async_raw", 1), ("weight_stashing", 1), ("two_buffered", 1),
                            ("optimizer_prediction", 1), ("gpipe", 4)):
            st = build_stages(build_layers(CONFIG1_DIMS, CONFIG1_ACTS), 4, torch_init(0, device), device=device)
            opts = [OptimizerState(OptimizerConfig("adam"), s.param_names, device=device) for s in st]
            g = GraphedExecute(build_timeline(strategy, 4, n_batches, t), st, opts, strategy, data, "softmax_xent",
                               lambda mb: 1e-4, warmup_runs=1, streams="stage")
            g.replay()
            torch.cuda.synchronize(device)
            graphs[strategy] = g
        times = {s: [] for s in graphs}
        for _ in range(trials):
            for s, g in graphs.items():
                times[s].append(_time_replays(torch, device, g, 1))
        out = {"config": f"config1 MLP {CONFIG1_DIMS}, B={BATCH}, Adam lr 1e-4, D=4 on 1 GPU, {n_batches} "
                         f"mini-batches per graphed run, one stream per stage, fp32; gpipe T=4"}
        for s, g in graphs.items():
            rep = g.report()
            out[s] = {"samples_per_s": round(n_batches * BATCH / statistics.median(times[s]), 1),
                      "snapshot_peaks": rep.snapshot_peaks, "final_loss": rep.losses[-1]}
        return out
    finally:
        graphs = None
        torch.cuda.empty_cache()
