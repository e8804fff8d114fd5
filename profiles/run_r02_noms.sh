# lane256 without the requests-in-rank-order array (1 KB smaller slot; scans read s_mem[s_por[r]]) vs the in-tree.
mkdir -p gpurun_out
exec > gpurun_out/noms_ab.txt 2>&1
SGPU_LIB=$PWD/build_ab/libsgpu_noms.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_noms.log 2>&1; echo "pytest noms rc=$?"; tail -2 gpurun_out/pytest_gpu_noms.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in noms tree; do
  lib=""; [ "$v" = "noms" ] && lib="$PWD/build_ab/libsgpu_noms.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
