#!/bin/bash
# Round-1 profile captures (run on a B200 through gpurun, one GPU):
#   launch list of one render frame (+ warm-up frames) and full-set captures of
#   the render kernels, then the same for three C3 train steps.
# Each command runs once without ncu first (exit 0 required), as the profiling
# recipe asks; outputs land in gpurun_out/ and the summaries are copied here.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-train --no-cpu-baseline"
$CMD > gpurun_out/plain_render.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_decode|k_traverse_bfs|k_composite" -s 5 -c 5 \
    -o gpurun_out/prof_render $CMD > /dev/null 2>&1
TCMD="python profiles/train_step_probe.py volumetric 3"
$TCMD > gpurun_out/plain_train.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train.csv $TCMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_fwd_in_t|k_fwd_mid|k_bwd_feat|k_loss|k_adam|k_bias_relu" \
    -s 7 -c 7 -o gpurun_out/prof_train $TCMD > /dev/null 2>&1
# the same three steps with the 3xTF32 tensor-core GEMMs (gemm_x3.cu)
XCMD="python profiles/train_step_probe.py volumetric 3 tf32x3"
$XCMD > gpurun_out/plain_train_x3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_x3.csv $XCMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_bwd_feat|k_fwd_in_t|k_fwd_mid" \
    -s 9 -c 9 -o gpurun_out/prof_train_x3 $XCMD > /dev/null 2>&1
