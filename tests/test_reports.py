"""Run-output formats (report.json / losses.csv / versions.csv) byte-compatible
with the reference's writers (experiments.py:305-392). CPU only: the
VersionRecords come from the oracle run of the same config (records are
timeline-determined), losses from the reference's own file."""

import json
from pathlib import Path

import numpy as np

from oracle import data_ref, optim_ref, rng_ref, runtime_ref
from paper_2312_00839_b200.reports import (
    LOSS_CSV_HEADER,
    VERSIONS_CSV_HEADER,
    config_hash,
    csv_text,
    json_text,
    loss_rows,
    run_report_obj,
    version_rows,
    write_run_outputs,
)
from paper_2312_00839_b200.runtime import RunReport, VersionRecord
from paper_2312_00839_b200.schedule import bubble_ratio, build_1f1b, makespan, steady_state_window

FILES = Path(__file__).resolve().parent / "golden" / "files"


def oracle_report():
    cfg = json.loads((FILES / "config.json").read_text())
    d = cfg["dataset"]
    xt, yt, _, _, loss = data_ref.make_dataset(d["kind"], d["n_samples"], d["seed"], input_dim=d["input_dim"],
                                               target_dim=d["target_dim"], noise=d["noise"])
    batches = data_ref.Batches(xt, yt, cfg["training"]["batch_size"])
    n = cfg["training"]["n_epochs"] * batches.steps_per_epoch
    out = runtime_ref.run(cfg["model"]["layer_dims"], cfg["model"]["activations"], cfg["depth"], n, cfg["strategy"],
                          optim_ref.Hyper("adam"), batches.batch, loss, lambda mb: cfg["training"]["lr"],
                          lambda i, a, b: rng_ref.layer_init(cfg["seed"], i, a, b))
    ref_losses = [float(line.split(",")[2]) for line in (FILES / "losses.csv").read_text().split("\n")[1:] if line]
    tl = build_1f1b(cfg["depth"], n)
    steady = steady_state_window(tl)
    rep = RunReport(
        strategy=cfg["strategy"], timeline_kind="1f1b", depth=cfg["depth"], n_batches=n, micro_per_mini=1,
        losses=ref_losses,
        records=[VersionRecord(*r[:3], *r[3:]) for r in out["records"]],
        snapshot_peaks=out["snapshot_peaks"], stash_peaks=out["stash_peaks"], final_versions=out["final_versions"],
        params_checksum="x", bubble_overall=str(bubble_ratio(tl)), bubble_steady=str(bubble_ratio(tl, *steady)),
        steady_window=steady, makespan_unit=makespan(tl),
    )
    return cfg, rep, batches.steps_per_epoch, out


def test_versions_and_losses_csv_byte_identical():
    cfg, rep, spe, out = oracle_report()
    assert np.allclose(out["losses"], rep.losses, rtol=0, atol=0)  # the oracle reproduces the reference
    assert csv_text(VERSIONS_CSV_HEADER.split(","), version_rows(rep)) == (FILES / "versions.csv").read_text()
    assert csv_text(LOSS_CSV_HEADER.split(","), loss_rows(rep, spe)) == (FILES / "losses.csv").read_text()


def test_report_json_matches_reference_fields():
    cfg, rep, spe, _ = oracle_report()
    want = json.loads((FILES / "report.json").read_text())
    got = run_report_obj(rep, config=cfg, seed=want["seed"], last_epoch_loss=want["last_epoch_loss"],
                         eval_loss=want["eval_loss"], eval_accuracy=want["eval_accuracy"])
    assert got["config_hash"] == want["config_hash"] == config_hash(cfg)
    for k in want:
        if k != "params_checksum":  # hashes fp64 bytes in the reference, fp32 here
            assert got[k] == want[k], k
    assert json_text(got).startswith("{\n  ")


def test_write_run_outputs(tmp_path):
    cfg, rep, spe, _ = oracle_report()
    d = write_run_outputs(rep, tmp_path / "out", spe, config=cfg)
    assert (d / "versions.csv").read_text() == (FILES / "versions.csv").read_text()
    d2 = write_run_outputs(rep, tmp_path / "outj", spe, fmt="json", config=cfg)
    assert json.loads((d2 / "losses.json").read_text())[0]["mb"] == 1
