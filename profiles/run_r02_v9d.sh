# lane256 resident warps (8 / 10 / 12 per SM) on C3 at HEAD -> gpurun_out/v9d.txt
mkdir -p gpurun_out
exec > gpurun_out/v9d.txt 2>&1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms')" "$@"; }
run() { if [ "$1" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$1.so"; fi
  SGPU_LIB=$lib timeout 600 python bench.py --config $2 --steps $3 --warmup 2 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $1 $2 || tail -3 gpurun_out/mv.err; }
for i in 1 2 3; do for v in tree l256mb5 l256mb6; do run $v C3 3; done; done
