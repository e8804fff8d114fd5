# lane256 speculative fit lookup (fit-table row, rank->position word and the
# next request loaded with the bucket entry's rank): in-tree vs
# build_ab/libsgpu_head.so (packed buckets), C3 interleaved.
mkdir -p gpurun_out
exec > gpurun_out/spec_ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2 3; do for v in tree head; do
  lib=""; [ "$v" = "head" ] && lib="$PWD/build_ab/libsgpu_head.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
