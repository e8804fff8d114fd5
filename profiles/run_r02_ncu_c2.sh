# One ncu --set full capture of the C2 K1 launch (main pass) -> gpurun_out/r02_c2_<tag>.ncu-rep
mkdir -p gpurun_out
TAG=${TAG:-head}
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -c 1 -k regex:trace_sim_lane_kernelILi2ELb0 -s 3 -o gpurun_out/r02_c2_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2_$TAG.log 2>&1; echo "ncu rc=$?"
python profiles/ncu_summary.py gpurun_out/r02_c2_$TAG.ncu-rep
