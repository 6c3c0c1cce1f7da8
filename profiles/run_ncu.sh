#!/usr/bin/env bash
# Profiling recipe (B200_PROFILING.md), run on the GPU box from the repo root:
#   1. the command once without ncu (must exit 0),
#   2. the launch list of the same command (cold-cache, serialised: compare shares),
#   3. one `--set full` capture of the dominant kernel (temporally blocked sweep).
set -u
CMD="python bench.py --steps 4 --warmup 3 --no-cpu --e2e-steps 0 ${BENCH_ARGS:-}"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:block_kernel -s ${NCU_SKIP:-30} -c ${NCU_COUNT:-1} \
    -o gpurun_out/prof_block $CMD > gpurun_out/ncu_full.log 2>&1
echo done
