# lane256 with whole 16-byte records (arrival, request, busy word) per
# position vs the in-tree (request, busy) pairs + separate arrivals.
mkdir -p gpurun_out
exec > gpurun_out/rs4_ab.txt 2>&1
SGPU_LIB=$PWD/build_ab/libsgpu_rs4.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rs4 rc=$?"; tail -2 gpurun_out/pytest_gpu.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in rs4 tree; do
  lib=""; [ "$v" = "rs4" ] && lib="$PWD/build_ab/libsgpu_rs4.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
