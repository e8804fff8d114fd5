# lane256 with an 16-stride fit table (1 KB smaller slot, up to 7 extra rank
# lookups from one 16-byte rank -> position load) vs the in-tree 4-stride.
mkdir -p gpurun_out
exec > gpurun_out/fs16_ab.txt 2>&1
SGPU_LIB=$PWD/build_ab/libsgpu_fs16.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_fs16.log 2>&1; echo "pytest fs16 rc=$?"; tail -2 gpurun_out/pytest_gpu_fs16.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in fs16 tree; do
  lib=""; [ "$v" = "fs16" ] && lib="$PWD/build_ab/libsgpu_fs16.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
