cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/sw.log
python profiles/sweep_bench.py --T 4,5,6,7,8 >> gpurun_out/sw.log 2>&1
python profiles/sweep_bench.py --variant nag --T 5 >> gpurun_out/sw.log 2>&1
python profiles/fns_time.py >> gpurun_out/sw.log 2>&1
