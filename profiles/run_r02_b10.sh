# C2 at ten two-warp blocks per SM (20 warps; 8-stride fit table, 32
# buckets: 10.9 KB per warp) vs the in-tree nine-block 4-stride build.
mkdir -p gpurun_out
exec > gpurun_out/b10_ab.txt 2>&1
SGPU_LIB=$PWD/build_ab/libsgpu_b10.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_b10.log 2>&1; echo "pytest b10 rc=$?"; tail -2 gpurun_out/pytest_gpu_b10.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2 3; do for v in b10 tree; do
  lib=""; [ "$v" = "b10" ] && lib="$PWD/build_ab/libsgpu_b10.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C2 || tail -3 gpurun_out/mv.err
done; done
