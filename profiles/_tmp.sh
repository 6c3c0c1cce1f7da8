cd $GRAFT_REPO_ROOT
echo base > gpurun_out/c1.log; python profiles/cfg1_probe.py 2>&1 | tail -2 >> gpurun_out/c1.log
for p in 4096 2048 1024 512 256; do echo "1024 threads, points/CTA $p" >> gpurun_out/c1.log; RICHGPU_LIB=paper_2412_08076_b200/librg_cl1024.so RG_CL_POINTS=$p python profiles/cfg1_probe.py 2>&1 | tail -2 >> gpurun_out/c1.log; done
