# Loop-free bucket fill (C2 A/B vs HEAD), lane256 working set: per-warp rank
# scratch, 6/8/10 warps per SM, 8 traces per warp (C3) -> gpurun_out/v9c.txt
mkdir -p gpurun_out
exec > gpurun_out/v9c.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms')" "$@"; }
run() { if [ "$1" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$1.so"; fi
  SGPU_LIB=$lib timeout 600 python bench.py --config $2 --steps $3 --warmup 2 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $1 $2 || tail -3 gpurun_out/mv.err; }
for i in 1 2 3; do for v in tree old; do run $v C2 5; done; done
for i in 1 2; do for v in tree old l256mb3 l256mb5 l256g8; do run $v C3 3; done; done
