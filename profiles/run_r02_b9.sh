# C2 at 9 two-warp blocks per SM (18 warps; 4-stride fit table, 128 buckets:
# 12.2 KB per warp) vs the in-tree 8-block 2-stride build, interleaved.
mkdir -p gpurun_out
exec > gpurun_out/b9_ab.txt 2>&1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
SGPU_LIB=$PWD/build_ab/libsgpu_b9.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2
for i in 1 2 3; do for v in tree b9; do
  lib=""; [ "$v" = "b9" ] && lib="$PWD/build_ab/libsgpu_b9.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C2 || tail -3 gpurun_out/mv.err
done; done
