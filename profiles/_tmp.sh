cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/refresh2.log
python profiles/configs_bench.py --only 5 --out gpurun_out/configs5.json > gpurun_out/configs5.log 2>&1; echo configs=$? >> gpurun_out/refresh2.log
