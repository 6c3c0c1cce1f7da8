cd $GRAFT_REPO_ROOT
echo "== base" > gpurun_out/sw.log; python profiles/sweep_bench.py --T 4,5,6 >> gpurun_out/sw.log 2>&1
for L in librg_c128 librg_r128; do echo "== $L" >> gpurun_out/sw.log; RICHGPU_LIB=paper_2412_08076_b200/$L.so python profiles/sweep_bench.py --T 3,4,5,6,7,8 >> gpurun_out/sw.log 2>&1; done
