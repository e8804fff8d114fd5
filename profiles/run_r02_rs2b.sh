# lane256 interleaved pairs at 6 blocks/SM (register cap 168) vs HEAD.
mkdir -p gpurun_out
exec > gpurun_out/rs2b_ab.txt 2>&1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in rs2mb6 h2; do
  lib="$PWD/build_ab/libsgpu_$v.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
