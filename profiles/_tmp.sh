cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_reference_contracts.py -q > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
