# Round-1 evidence for the K1 lane kernel on C2 (one GPU):
#   1. launch list of the bench command (gpu__time_duration per launch)
#   2. one --set full capture of the K1 lane kernel (source-attributed)
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trace_sim_lane -s 3 -c 1 -o gpurun_out/lane_full python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/lane_full.log 2>&1; echo "ncu full rc=$?"
