# A/B on one GPU: gpu tests on the in-tree build, then the kernel-only bench
# line of the in-tree build against build_ab/libsgpu_old.so (previous commit).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for i in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_new.json 2> gpurun_out/bench_new.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_new.json'));print('new',d['value'],d['ms_per_step'])"
SGPU_LIB=$PWD/build_ab/libsgpu_old.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_old.json 2> gpurun_out/bench_old.err; echo "bench old rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_old.json'));print('old',d['value'],d['ms_per_step'])"
done
tail -3 gpurun_out/bench_new.err
