cd $GRAFT_REPO_ROOT
python profiles/vcycle_levels.py > gpurun_out/vc.log 2>&1
RG_CB9_MINSIDE=200 python profiles/vcycle_levels.py >> gpurun_out/vc.log 2>&1
RG_CB9_MINSIDE=100 python profiles/vcycle_levels.py >> gpurun_out/vc.log 2>&1
