# ncu --set full capture of the DST line kernel (source of profiles/ncu_dst_r01.json)
cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:dst_lines_kernel -s 6 -c 2 \
    -o gpurun_out/prof_dst python profiles/fns_time.py > gpurun_out/ncu_dst.log 2>&1
echo done
