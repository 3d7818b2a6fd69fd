"""Wire/file formats of a run, byte-compatible with the
reference's writers (pkg/src/pipesim/experiments.py:305-392): `losses.csv`
(mb,epoch,loss), `versions.csv` (VersionRecords sorted by (mb, micro,
stage)), JSON with indent 2 and sorted keys, and the canonical-JSON config
hash used to name output directories (config.py:293-298).
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

from .runtime import RunReport, memory_peaks, staleness_and_inconsistency

LOSS_CSV_HEADER = "mb,epoch,loss"
VERSIONS_CSV_HEADER = (
    "mb,micro,stage,forward_version,predicted,prediction_target,"
    "backward_version,live_backward_version,staleness,inconsistent"
)


def cell(v) -> str:
    """One CSV cell: '' for None, 1/0 for bools, repr for floats, '|'-joined lists."""
    if v is None:
        return ""
    if isinstance(v, bool):
        return "1" if v else "0"
    if isinstance(v, float):
        return repr(v)
    if isinstance(v, (list, tuple)):
        return "|".join(str(x) for x in v)
    return str(v)


def csv_text(columns: list[str], rows: list[dict]) -> str:
    out = [",".join(columns)]
    out += [",".join(cell(r.get(c)) for c in columns) for r in rows]
    return "\n".join(out) + "\n"


def json_text(obj) -> str:
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


def loss_rows(report: RunReport, steps_per_epoch: int) -> list[dict]:
    return [{"mb": mb, "epoch": (mb - 1) // steps_per_epoch + 1, "loss": float(loss)}
            for mb, loss in enumerate(report.losses, start=1)]


def version_rows(report: RunReport) -> list[dict]:
    return [r.to_dict() for r in sorted(report.records, key=lambda r: (r.mb, r.micro, r.stage))]


def canonical_json(cfg: dict) -> str:
    return json.dumps(cfg, sort_keys=True, separators=(",", ":"))


def config_hash(cfg: dict) -> str:
    return hashlib.sha256(canonical_json(cfg).encode()).hexdigest()[:12]


def run_report_obj(report: RunReport, *, config: dict | None = None, seed=None, final_loss=None,
                   last_epoch_loss=None, eval_loss=None, eval_accuracy=None) -> dict:
    """report.json body (experiments.py:346-372)."""
    info = staleness_and_inconsistency(report)
    return {
        "config": config,
        "config_hash": config_hash(config) if config is not None else None,
        "seed": seed,
        "strategy": report.strategy,
        "schedule": report.timeline_kind,
        "depth": report.depth,
        "n_batches": report.n_batches,
        "micro_per_mini": report.micro_per_mini,
        "final_loss": final_loss if final_loss is not None else report.losses[-1],
        "last_epoch_loss": last_epoch_loss,
        "eval_loss": eval_loss,
        "eval_accuracy": eval_accuracy,
        "inconsistent_total": info["inconsistent_total"],
        "mean_staleness": info["mean_staleness"],
        "per_stage": info["per_stage"],
        "memory_peaks": memory_peaks(report),
        "activation_stash_peaks": report.stash_peaks,
        "final_versions": report.final_versions,
        "params_checksum": report.params_checksum,
        "bubble_overall": report.bubble_overall,
        "bubble_steady": report.bubble_steady,
        "steady_window": list(report.steady_window) if report.steady_window else None,
        "makespan_unit": report.makespan_unit,
    }


def write_run_outputs(report: RunReport, out_dir: Path, steps_per_epoch: int, fmt: str = "csv",
                      **report_fields) -> Path:
    """report.json + losses/versions as csv or json (experiments.py:375-392)."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    (out_dir / "report.json").write_text(json_text(run_report_obj(report, **report_fields)))
    losses, versions = loss_rows(report, steps_per_epoch), version_rows(report)
    if fmt == "json":
        (out_dir / "losses.json").write_text(json_text(losses))
        (out_dir / "versions.json").write_text(json_text(versions))
    else:
        (out_dir / "losses.csv").write_text(csv_text(LOSS_CSV_HEADER.split(","), losses))
        (out_dir / "versions.csv").write_text(csv_text(VERSIONS_CSV_HEADER.split(","), versions))
    return out_dir


DEVICE_TIMELINE_CSV_HEADER = "stage,kind,mb,micro,start_us,end_us"


def write_device_timeline(report: RunReport, path: Path) -> Path:
    """`device_timeline.csv` of a traced run (execute(..., trace=True)): one
    row per executed event in the reference's event order, with its start
    and end on the device clock (µs from the run's first event) — the
    measured counterpart of the slot timeline (schedule.timeline_csv_text)."""
    rows = getattr(report, "device_timeline", None)
    if rows is None:
        raise ValueError("the report has no device_timeline: run execute(..., trace=True)")
    path = Path(path)
    path.write_text(csv_text(DEVICE_TIMELINE_CSV_HEADER.split(","), rows))
    return path
