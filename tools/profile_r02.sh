#!/bin/bash
# Round-2 profiling call on the GPU box: plain short bench (must exit 0), the ncu launch list of the same
# command, one full capture of the step's main kernels, one of the k = 1 kernels.  Usage (under gpurun):
#   bash tools/profile_r02.sh OUTDIR
set -u
OUT=${1:-gpurun_out/prof}
mkdir -p "$OUT"
CMD="python bench.py --steps 3 --warmup 3 --reps 1 --no-small --no-cpu-baseline --affine-steps 0 --fine-steps 0 --e2e-steps 1 --no-offline --k1-steps 0"
$CMD > "$OUT/plain.log" 2>&1 || { echo "plain bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file "$OUT/launches.csv" $CMD > "$OUT/ncu_list.log" 2>&1
echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k regex:"k_pcg_tm|k_flux_transport|k_project|k_transform_h|k_block_chol|k_recon|k_ns_gemm_tc|k_coarse_rt_s|k_hist" -s 30 -c 14 -o "$OUT/prof" $CMD > "$OUT/ncu_full.log" 2>&1
echo "full capture exit $?"
CMD1="python bench.py --steps 2 --warmup 3 --reps 1 --no-small --no-cpu-baseline --affine-steps 0 --fine-steps 0 --e2e-steps 1 --no-offline --k1-steps 2 --basis poly"
ncu --set full --clock-control none --import-source on -k regex:"k1_" -s 12 -c 5 -o "$OUT/prof_k1" $CMD1 > "$OUT/ncu_k1.log" 2>&1
echo "k1 capture exit $?"
