"""How much of config 1's single-GPU prediction overhead is K3's W_hat store?
Builds (here, `--build`) a probe copy of the whole library with
-DPO_PROBE_K3_NO_WHAT (K3 skips the W_hat store: the forwards then read a
stale staging buffer, so the numbers are timing only), and on the box times
the graphed stage-concurrent config-1 run, prediction on/off, with the shipped
library and with the probe library (separate processes).

  python scripts/k3_no_what_probe.py --build
  python scripts/k3_no_what_probe.py [--probe]
"""
import argparse
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
PROBE_DIR = ROOT / "paper_2312_00839_b200" / "build" / "probe"
PROBE = PROBE_DIR / "libpipeoptim_no_what.so"

ap = argparse.ArgumentParser()
ap.add_argument("--build", action="store_true")
ap.add_argument("--define", default="PO_PROBE_K3_NO_WHAT", help="probe macro (build); the library name follows it")
ap.add_argument("--probe", action="store_true")
a = ap.parse_args()
if a.build:
    from paper_2312_00839_b200 import build as b

    PROBE = PROBE_DIR / ("libpipeoptim_no_what.so" if a.define == "PO_PROBE_K3_NO_WHAT" else
                         f"libpipeoptim_{a.define.lower()}.so")
    cut = b.cutlass_root()
    objs = []
    PROBE.parent.mkdir(parents=True, exist_ok=True)
    for src in b.sources(cut):
        obj = PROBE.parent / (src.stem + "_" + a.define.lower() + ".o")
        extra = b._cutlass_include(cut) if src.name == b.GEMM_TU else []
        cmd = [b.nvcc_path(), *b.ARCH_FLAGS, *b.NVCC_FLAGS, f"-I{b.INCLUDE}", *extra, f"-D{a.define}", "-c",
               "-o", str(obj), str(src)]
        if src.suffix == ".cpp":
            cmd[1:1] = ["-x", "cu"]
        objs.append((obj, subprocess.Popen(cmd)))
    assert all(p.wait() == 0 for _, p in objs)
    subprocess.run([b.nvcc_path(), *b.ARCH_FLAGS, "-shared", "-o", str(PROBE), *[str(o) for o, _ in objs], "-lcuda"],
                   check=True)
    sys.exit(0)

import torch  # noqa: E402

from paper_2312_00839_b200 import _lib  # noqa: E402

if a.probe:
    _lib._lib = _lib.load(PROBE)
from paper_2312_00839_b200 import bench_pipeline as bp  # noqa: E402

dev = torch.device("cuda", 0)
r = bp.single_gpu_pipeline(torch, dev, n_batches=64, with_eager=False, with_roofline=False)
print(json.dumps({"lib": "probe_no_what" if a.probe else "shipped", "pred_off": r["pred_off"]["samples_per_s"],
                  "pred_on": r["pred_on"]["samples_per_s"], "overhead": r["prediction_overhead"]}), flush=True)
