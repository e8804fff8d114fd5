# Output-row prewrite (coalesced SG_NEVER stores of the group's grant / end
# rows before the lanes' per-app stores): in-tree vs build_ab/libsgpu_cur.so,
# C2/C4/C5 interleaved, GPU tests, and the DRAM bytes of one C2 main-pass
# launch of each build.
mkdir -p gpurun_out
exec > gpurun_out/prewrite_ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
show() { python -c "import json,sys;d=json.load(open(sys.argv[1]));print(sys.argv[2],sys.argv[3],round(d['value']/1e6,3),'M',round(d['ms_per_step'],3),'ms',d['clocks']['sm_mhz'])" "$@"; }
for i in 1 2 3; do for v in tree cur; do
  lib=""; [ "$v" = "cur" ] && lib="$PWD/build_ab/libsgpu_cur.so"
  for c in C2 C4 C5; do
  SGPU_LIB=$lib timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/mv.json 2> gpurun_out/mv.err && show gpurun_out/mv.json $v $c || tail -3 gpurun_out/mv.err
  done
done; done
for v in tree cur; do
  lib=""; [ "$v" = "cur" ] && lib="$PWD/build_ab/libsgpu_cur.so"
  SGPU_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:trace_sim_lane_kernelILi2ELb0 -s 3 -c 1 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/$v /"
done
