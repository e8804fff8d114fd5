# Output-row prewrite issued before the group's staging (stores overlap the
# staging loads) vs after it (in-tree), C2 interleaved.
mkdir -p gpurun_out
exec > gpurun_out/pw0_ab.txt 2>&1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2 3; do for v in pw0 tree; do
  lib=""; [ "$v" = "pw0" ] && lib="$PWD/build_ab/libsgpu_pw0.so"
  SGPU_LIB=$lib timeout 600 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C2 || tail -3 gpurun_out/mv.err
done; done
