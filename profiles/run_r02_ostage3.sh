# Grant/end staging copy-out variants: in-tree (out-of-line batched copy) vs
# build_ab/libsgpu_v1r.so (inline row copy, restrict + unroll 4) vs
# build_ab/libsgpu_old.so (no staging), C2/C4/C5 interleaved.
mkdir -p gpurun_out
exec > gpurun_out/ostage3_ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2; do for v in tree v1r old; do
  if [ "$v" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$v.so"; fi
  for c in C2 C4 C5; do
  SGPU_LIB=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v $c || tail -3 gpurun_out/mv.err
  done
done; done
