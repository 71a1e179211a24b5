#!/bin/bash
# Round-2 end-of-round profile captures of the render path (B200 via gpurun, one GPU),
# after the decoder-head, traversal-origin, two-phase device frame and sparse host-frame
# changes. Each command first runs once without ncu (exit 0 required); outputs in
# gpurun_out/, summaries written to profiles/ by profiles/summarize.py.
#   render:   the bench's C2 headline frame (launch list + full set of the top kernels)
#   render20: the 20-object C2' frame (same)
# The train kernels are unchanged since the r2c captures (profiles/r2c_train.*).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-train --no-cpu-baseline --headline-only"
$CMD > gpurun_out/plain_render_d.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render_d.csv $CMD > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_decode|k_traverse_bfs|k_composite|k_pack_fg" -s 5 -c 6 \
    -o gpurun_out/prof_render_d $CMD > /dev/null 2>&1
CMD20="python bench.py --steps 2 --warmup 3 --no-train --no-cpu-baseline --headline-only --objects 20"
$CMD20 > gpurun_out/plain_render20_d.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_render20_d.csv $CMD20 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_decode|k_traverse_bfs|k_composite" -s 5 -c 5 \
    -o gpurun_out/prof_render20_d $CMD20 > /dev/null 2>&1
