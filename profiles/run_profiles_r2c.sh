#!/bin/bash
# Round-2 (final) profile captures (B200 via gpurun, one GPU). Each command first runs
# once without ncu (exit 0 required), as the profiling recipe asks; outputs in
# gpurun_out/, summaries copied to profiles/ by profiles/summarize.py.
#   render: the bench's C2 headline frame (launch list + full set of the top kernels)
#   render20: the 20-object C2' frame (same)
#   train:  three C3 train steps (default fp32-accurate 3xTF32 GEMMs, graph replay)
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-train --no-cpu-baseline --headline-only"
$CMD > gpurun_out/plain_render_c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render_c.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_decode|k_traverse_bfs|k_composite" -s 5 -c 5 \
    -o gpurun_out/prof_render_c $CMD > /dev/null 2>&1
CMD20="python bench.py --steps 2 --warmup 3 --no-train --no-cpu-baseline --headline-only --objects 20"
$CMD20 > gpurun_out/plain_render20_c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render20_c.csv $CMD20 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_decode|k_traverse_bfs|k_composite" -s 5 -c 5 \
    -o gpurun_out/prof_render20_c $CMD20 > /dev/null 2>&1
TCMD="python profiles/train_step_probe.py volumetric 3"
$TCMD > gpurun_out/plain_train_c.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_train_c.csv $TCMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_gemm|k_bwd_feat|k_fwd_in_t|k_fwd_mid|k_adam|k_dw_reduce|k_bwd_head_c" -s 16 -c 16 \
    -o gpurun_out/prof_train_c $TCMD > /dev/null 2>&1
