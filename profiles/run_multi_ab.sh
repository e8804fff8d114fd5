# Kernel-only C2 bench of the in-tree build and of every build_ab/libsgpu_<v>.so
# named in VARIANTS, interleaved N_AB times; then CONFIGS once each.
# Output -> gpurun_out/multi_ab.txt
mkdir -p gpurun_out
exec > gpurun_out/multi_ab.txt 2>&1
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,2),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
run() {  # variant config steps
  if [ "$1" = "tree" ]; then lib=""; else lib="$PWD/build_ab/libsgpu_$1.so"; fi
  SGPU_LIB=$lib timeout 600 python bench.py --config $2 --steps $3 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $1 $2 || tail -3 gpurun_out/mv.err
}
for i in $(seq ${N_AB:-3}); do for v in tree $VARIANTS; do run $v C2 5; done; done
for c in ${CONFIGS:-C4 C5}; do for v in tree $VARIANTS; do run $v $c 3; done; done
