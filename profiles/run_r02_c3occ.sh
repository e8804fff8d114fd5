# C3 lane256 occupancy A/B: the in-tree build (occupancy-limited, 6 blocks
# = 12 warps/SM) against builds capped at 3/4/5 blocks per SM, interleaved.
mkdir -p gpurun_out
exec > gpurun_out/c3occ_ab.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],round(d['value']/1e6,3),'M',round(d['ms_per_step'],2),'ms')" "$@"; }
for i in 1 2; do for v in tree c3b3 c3b4 c3b5; do
  if [ "$v" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$v.so"; fi
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v || tail -3 gpurun_out/mv.err
done; done
