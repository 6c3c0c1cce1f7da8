cd $GRAFT_REPO_ROOT
python profiles/vcycle_levels.py > gpurun_out/vc.log 2>&1
RG_PS_MAX=4096 python profiles/vcycle_levels.py >> gpurun_out/vc.log 2>&1
