# lane256 rank lookup: buckets 128/256/512, sorted-request table on/off -> gpurun_out/v9b.txt
mkdir -p gpurun_out
exec > gpurun_out/v9b.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "octet or C3 or shapes or golden" 2>&1 | tail -1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms')" "$@"; }
run() { if [ "$1" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$1.so"; fi
  SGPU_LIB=$lib timeout 600 python bench.py --config $2 --steps $3 --warmup 2 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $1 $2 || tail -3 gpurun_out/mv.err; }
for i in 1 2 3; do for v in tree l256lb128 l256nosort l256lb512; do run $v C3 3; done; done
