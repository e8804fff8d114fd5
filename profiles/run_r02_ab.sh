# A/B on one GPU: the GPU tests on the in-tree build, then the kernel-only
# bench lines of the in-tree build against build_ab/libsgpu_old.so
# (profiles/build_ab_lib.sh), interleaved, for C2 (N_AB times) and once for
# each of CONFIGS (default "C4 C5").  Output -> gpurun_out/ab.txt.
mkdir -p gpurun_out
exec > gpurun_out/ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
[ -n "$NO_TESTS" ] || { timeout 1200 python -m pytest tests -m gpu -x -q ${TESTS_K:+-k "$TESTS_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log; }
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],d['value'],d['ms_per_step'],d['clocks']['sm_mhz'])" "$@"; }
for i in $(seq ${N_AB:-3}); do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bn.json 2> gpurun_out/bn.err; show gpurun_out/bn.json new C2
  SGPU_LIB=$PWD/build_ab/libsgpu_old.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bo.json 2> gpurun_out/bo.err; show gpurun_out/bo.json old C2
done
for c in ${CONFIGS:-C4 C5}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bn.json 2> gpurun_out/bn.err; show gpurun_out/bn.json new $c
  SGPU_LIB=$PWD/build_ab/libsgpu_old.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/bo.json 2> gpurun_out/bo.err; show gpurun_out/bo.json old $c
done
