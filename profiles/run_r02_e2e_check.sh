# End-to-end C2 (sg_simulate_batch_host) box check: in-tree (HEAD) vs
# build_ab/libsgpu_old.so (58d8b56, the previous evidence commit), interleaved.
mkdir -p gpurun_out
exec > gpurun_out/e2e_check.txt 2>&1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],'kernel',round(d['value']/1e6,1),'M e2e',round(d['e2e']['value']/1e6,1),'M')" "$@"; }
for i in 1 2 3; do for v in tree old; do
  lib=""; [ "$v" = "old" ] && lib="$PWD/build_ab/libsgpu_old.so"
  SGPU_LIB=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v || tail -3 gpurun_out/mv.err
done; done
