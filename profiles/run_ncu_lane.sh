set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:trace_sim_lane_kernelILi2ELb0 -s 3 -c 1 -o gpurun_out/lane_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/lane_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/lane_full.log
