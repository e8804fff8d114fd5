# Grant/end row staging A/B (C2: in-tree build vs build_ab/libsgpu_old.so,
# HEAD without staging), C3 lane256 register-cap variants, then one ncu
# --set full capture of the C2 main-pass kernel of the in-tree build.
mkdir -p gpurun_out
exec > gpurun_out/ostage_ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2 3; do for v in tree old; do
  if [ "$v" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$v.so"; fi
  for c in C2 C4 C5; do
  SGPU_LIB=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v $c || tail -3 gpurun_out/mv.err
  done
done; done
for i in 1 2; do for v in tree c3mb7 c3mb8; do
  if [ "$v" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$v.so"; fi
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
TAG=ostage bash profiles/run_r02_ncu_c2.sh
