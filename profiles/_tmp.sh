cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/c1.log
python profiles/cfg1_probe.py >> gpurun_out/c1.log 2>&1
