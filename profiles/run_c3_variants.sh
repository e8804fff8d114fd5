mkdir -p gpurun_out
exec > gpurun_out/multi_ab.txt 2>&1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],2),'ms')" "$@"; }
for i in 1 2; do for v in tree ofs2 oslot3; do
  if [ "$v" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$v.so"; fi
  SGPU_LIB=$lib timeout 600 python bench.py --config C3 --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v C3 || tail -3 gpurun_out/mv.err
done; done
SGPU_LIB=$PWD/build_ab/libsgpu_oslot3.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "octet" 2>&1 | tail -1
SGPU_LIB=$PWD/build_ab/libsgpu_ofs2.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "octet" 2>&1 | tail -1
