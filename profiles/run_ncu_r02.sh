#!/usr/bin/env bash
# Round-2 profiling recipe (B200_PROFILING.md), run on the GPU box from the repo root:
#   1. the bench command once without ncu (must exit 0),
#   2. the launch list of the same command (cold-cache, serialised: compare shares),
#   3. `--set full` captures of the kernels changed this round: the cluster
#      SOR wavefront (tri_kernel) and the pairwise MGS (mgs_persist_kernel).
set -u
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --e2e-steps 0 --no-configs"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_r02.csv $CMD > gpurun_out/ncu_launches.log 2>&1
python profiles/tri_ncu.py > /dev/null && ncu --set full --clock-control none --import-source on -k regex:tri_kernel -s 2 -c 1 \
    -o gpurun_out/prof_tri_r02_final python profiles/tri_ncu.py > gpurun_out/ncu_tri.log 2>&1
python profiles/mgs_ncu.py > /dev/null && ncu --set full --clock-control none --import-source on -k regex:mgs_persist -s 1 -c 1 \
    -o gpurun_out/prof_mgs_r02_final python profiles/mgs_ncu.py > gpurun_out/ncu_mgs.log 2>&1
echo done
