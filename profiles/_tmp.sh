cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/t.log
