#!/bin/bash
# Standalone probe builds of csrc/pipeoptim_gemm.cu with other tile shapes /
# stage carve-outs (scripts/gemm_tile_probe.py loads them by path; each also
# exports po_probe_gemm_smem). Output: scripts/_probe_libs/.
# Usage: build_gemm_tile_variants.sh N:K[:EXTRA_CARVEOUT_BYTES] ...
set -e
cd "$(dirname "$0")/.."
CUT=$(python -c "import sys; sys.path.insert(0,'.'); from paper_2312_00839_b200 import build as b; print(b.cutlass_root())")
OUT=scripts/_probe_libs
mkdir -p $OUT
rm -f $OUT/libgemm_*.so
for cfg in "$@"; do
  IFS=: read -r n k extra <<< "$cfg"
  extra=${extra:-0}
  tag=n${n}_k${k}_c${extra}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
    -diag-suppress 20012 -Iinclude -I$CUT/include -I$CUT/tools/util/include -DPO_PROBE_EXPORTS \
    -DPO_FASTF32_TILE_N=$n -DPO_FASTF32_TILE_K=$k -DPO_FASTF32_EXTRA_CARVEOUT=$extra -shared \
    -o $OUT/libgemm_$tag.so paper_2312_00839_b200/csrc/pipeoptim_gemm.cu > $OUT/build_$tag.log 2>&1 \
    || echo "build $tag failed" &
done
wait
ls $OUT/*.so
