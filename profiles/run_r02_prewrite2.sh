# Prewrite only for groups of >= 4 traces: in-tree vs build_ab/libsgpu_cur.so.
mkdir -p gpurun_out
exec > gpurun_out/prewrite2_ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in tree cur; do
  lib=""; [ "$v" = "cur" ] && lib="$PWD/build_ab/libsgpu_cur.so"
  for c in C2 C5; do
  SGPU_LIB=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v $c || tail -3 gpurun_out/mv.err
  done
done; done
