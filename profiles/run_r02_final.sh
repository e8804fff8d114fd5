# Round-2 evidence at HEAD in one gpurun call (all output -> gpurun_out/):
# GPU tests, smoke, one ncu --set full capture per configuration's K1 kernel
# (C2 first: it refreshes profiles/k1_traffic.json for the bench line), the
# bench line (C2, CPU reference beside it), the reference arm, the launch
# list of the bench command, C3-C5 lines, step programs, the 2-rank bench
# (gloo, one GPU) and the drop-in latency.
set -x
mkdir -p gpurun_out
lscpu > gpurun_out/lscpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base mangled -c 1"
timeout 600 $NCU -k regex:trace_sim_lane_kernelILi2ELb0 -s 3 -o gpurun_out/fin_c2 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
python profiles/update_traffic.py gpurun_out/fin_c2.ncu-rep
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
python profiles/summarize_launches.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1; cat gpurun_out/launches_summary.txt
timeout 1500 $NCU -k regex:trace_sim_lane256_kernel -s 2 -o gpurun_out/fin_c3 python bench.py --config C3 --steps 1 --warmup 2 --no-cpu --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 900 $NCU -k regex:trace_sim_lane_kernelILi4ELb0 -s 3 -o gpurun_out/fin_c4 python bench.py --config C4 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 rc=$?"
timeout 600 $NCU -k regex:trace_sim_lane_kernelILi2ELb0 -s 3 -o gpurun_out/fin_c5 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 600 $NCU -k regex:trace_prog_lane_kernel -s 2 -o gpurun_out/fin_prog python profiles/program_bench.py 262144 > gpurun_out/ncu_prog.log 2>&1; echo "ncu prog rc=$?"
python profiles/ncu_summary.py gpurun_out/fin_*.ncu-rep > gpurun_out/ncu_summary.md 2>&1; cat gpurun_out/ncu_summary.md
for c in C3 C4 C5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/other_$c.json 2> gpurun_out/other_$c.err; echo "$c rc=$?"; tail -c 300 gpurun_out/other_$c.json
done
timeout 300 python profiles/program_bench.py 262144 > gpurun_out/program_mode.txt 2>&1; cat gpurun_out/program_mode.txt
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; echo "2-rank rc=$?"; cat gpurun_out/bench_2rank.json
timeout 300 python profiles/dropin_latency.py > gpurun_out/dropin_latency.txt 2>&1; cat gpurun_out/dropin_latency.txt
