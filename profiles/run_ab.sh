# A/B on one GPU: gpu tests on the in-tree build, then the kernel-only bench
# line of the in-tree build against build_ab/libsgpu_old.so (profiles/build_ab_lib.sh),
# interleaved N_AB times (default 3), with each run's per-step K1 times.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ -n "$NO_TESTS" ] || { timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log; }
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],d['value'],d['ms_per_step'],d['clocks'])" "$@"; grep "per-step" "${1%.json}.err"; }
for i in $(seq ${N_AB:-3}); do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_new.json 2> gpurun_out/bench_new.err; show gpurun_out/bench_new.json new
SGPU_LIB=$PWD/build_ab/libsgpu_old.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_old.json 2> gpurun_out/bench_old.err; show gpurun_out/bench_old.json old
done
nvidia-smi
