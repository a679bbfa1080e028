#!/bin/bash
# One profiling call on the GPU box: debug-build timelines of the PCG and the projection, a plain short
# bench, then a full ncu capture of the step's main kernels.  Usage (under gpurun):
#   bash tools/profile_round.sh OUTDIR [kernel-regex]
set -u
OUT=${1:-gpurun_out/prof}
RE=${2:-"k_pcg_tm|k_flux_transport|k_project|k_transform_h"}
mkdir -p "$OUT"
if [ -f variants/debug.so ]; then
  LRBMS_LIB=variants/debug.so python tools/exp_timeline.py C5 > "$OUT/pcg_timeline.txt" 2>&1
  LRBMS_LIB=variants/debug.so python tools/exp_proj_phases.py C5 > "$OUT/proj_phases.txt" 2>&1
fi
CMD="python bench.py --steps 3 --warmup 3 --reps 1 --no-small --no-cpu-baseline --affine-steps 0 --fine-steps 0 --e2e-steps 1 --no-offline --k1-steps 0"
$CMD > "$OUT/plain.log" 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$RE" -s 8 -c 4 -o "$OUT/prof" $CMD > "$OUT/ncu.log" 2>&1
echo "ncu exit $?"
