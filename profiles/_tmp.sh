cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_parity.py -q -k "above_64" > gpurun_out/t.log 2>&1; echo rc=$? >> gpurun_out/t.log
