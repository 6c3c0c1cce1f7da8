cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? > gpurun_out/refresh.log
python profiles/configs_bench.py --out gpurun_out/configs.json > gpurun_out/configs.log 2>&1; echo configs=$? >> gpurun_out/refresh.log
bash profiles/run_ncu.sh >> gpurun_out/refresh.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/fns_launches.csv python profiles/fns_time.py > gpurun_out/ncu_fns.log 2>&1
python profiles/vcycle_levels.py > gpurun_out/vcycle_levels.json 2>&1
