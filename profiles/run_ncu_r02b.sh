#!/usr/bin/env bash
# `--set full` captures of the kernels of the last round-2 commits (each target
# runs once without ncu first); the reports are summarised on the box
# (profiles/summarize_ncu.py) because three reports exceed the 64 MiB that
# travel back.
set -u
mkdir -p gpurun_out /tmp/ncu
python profiles/tri_ncu.py > /dev/null && ncu --set full --clock-control none -k regex:tri_kernel -s 2 -c 1 \
    -o /tmp/ncu/tri python profiles/tri_ncu.py > gpurun_out/ncu_tri.log 2>&1
python profiles/mgs_ncu.py > /dev/null && ncu --set full --clock-control none -k regex:mgs_persist -s 1 -c 1 \
    -o /tmp/ncu/mgs python profiles/mgs_ncu.py > gpurun_out/ncu_mgs.log 2>&1
python profiles/fns_launch_target.py > /dev/null && ncu --set full --clock-control none \
    --profile-from-start off -k regex:"dstw_kernel|resid9_kernel" -c 4 \
    -o /tmp/ncu/fns python profiles/fns_launch_target.py > gpurun_out/ncu_fns.log 2>&1
for n in tri mgs fns; do python profiles/summarize_ncu.py full /tmp/ncu/$n.ncu-rep > gpurun_out/ncu_${n}_summary.json; done
echo done
