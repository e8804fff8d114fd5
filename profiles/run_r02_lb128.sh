# lane256 with 128 rank buckets (0.5 KB smaller slot) vs the in-tree 256.
mkdir -p gpurun_out
exec > gpurun_out/lb128_ab.txt 2>&1
SGPU_LIB=$PWD/build_ab/libsgpu_lb128.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_lb128.log 2>&1; echo "pytest lb128 rc=$?"; tail -2 gpurun_out/pytest_gpu_lb128.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in lb128 tree; do
  lib=""; [ "$v" = "lb128" ] && lib="$PWD/build_ab/libsgpu_lb128.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
