# In-tree 8-stride lane256 (two u64 loads of the rank -> position chunk):
# GPU tests, then C3 against build_ab/libsgpu_fs8.so (one uint4 load).
mkdir -p gpurun_out
exec > gpurun_out/fs8b.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in tree fs8; do
  lib=""; [ "$v" = "fs8" ] && lib="$PWD/build_ab/libsgpu_fs8.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 > gpurun_out/c3_$v.json 2> gpurun_out/mv.err && show gpurun_out/c3_$v.json $v C3 || tail -3 gpurun_out/mv.err
done; done
