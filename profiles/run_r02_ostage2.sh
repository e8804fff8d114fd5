# Grant/end row staging A/B, batched copy-out: in-tree build with staging
# (default) vs SGPU_OSTAGE=0 (direct per-app stores), C2/C4/C5 interleaved,
# then an ncu --set full capture of the C2 main-pass kernel.
mkdir -p gpurun_out
exec > gpurun_out/ostage2_ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2 3; do for v in 1 0; do
  for c in C2 C4 C5; do
  SGPU_OSTAGE=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json ostage=$v $c || tail -3 gpurun_out/mv.err
  done
done; done
TAG=ostage2 bash profiles/run_r02_ncu_c2.sh
