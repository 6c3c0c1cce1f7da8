cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/fns.log
python profiles/fns_time.py >> gpurun_out/fns.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/fns_launches.csv python profiles/fns_time.py > gpurun_out/ncu_fns.log 2>&1
