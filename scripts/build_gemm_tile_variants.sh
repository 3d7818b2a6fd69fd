#!/bin/bash
# Standalone probe builds of csrc/pipeoptim_gemm.cu with other tile shapes
# (scripts/gemm_tile_probe.py loads them by path). Output: scripts/_probe_libs/.
set -e
cd "$(dirname "$0")/.."
CUT=$(python -c "import sys; sys.path.insert(0,'.'); from paper_2312_00839_b200 import build as b; print(b.cutlass_root())")
OUT=scripts/_probe_libs
mkdir -p $OUT
for cfg in "$@"; do  # cfg = N:K, e.g. 128:32
  n=${cfg%%:*}; k=${cfg##*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -diag-suppress 20012 -Iinclude -I$CUT/include -I$CUT/tools/util/include \
    -DPO_FASTF32_TILE_N=$n -DPO_FASTF32_TILE_K=$k -shared -o $OUT/libgemm_n${n}_k${k}.so \
    paper_2312_00839_b200/csrc/pipeoptim_gemm.cu > $OUT/build_n${n}_k${k}.log 2>&1 &
done
wait
ls -la $OUT
