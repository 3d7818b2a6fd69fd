"""How much of po_wgrad_update's time is the in-kernel bf16x3 operand split?
Runs scripts/wgrad_kernel_bench.py against a probe library built with
-DPO_PROBE_NO_SPLIT (operands stored unsplit: wrong results, timing only):
  python scripts/k3_no_what_probe.py --build --define PO_PROBE_NO_SPLIT   # here
  python scripts/wgrad_split_probe.py                                      # box
"""
import ctypes, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2312_00839_b200 import _lib
_lib._lib = _lib.load(Path(__file__).resolve().parent.parent / "paper_2312_00839_b200/build/probe/libpipeoptim_po_probe_no_split.so")
import runpy
sys.argv = ["wgrad_kernel_bench.py"]
runpy.run_path(str(Path(__file__).resolve().parent / "wgrad_kernel_bench.py"), run_name="__main__")
