# One ncu --set full capture of the C3 K1 launch -> gpurun_out/r02_c3_<tag>.ncu-rep
mkdir -p gpurun_out
TAG=${TAG:-head}
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -c 1 -k regex:${KREGEX:-trace_sim_octet_kernel} -s 2 -o gpurun_out/r02_c3_$TAG python bench.py --config C3 --steps 1 --warmup 2 --no-cpu --no-e2e > gpurun_out/ncu_c3_$TAG.log 2>&1; echo "ncu rc=$?"
python profiles/ncu_summary.py gpurun_out/r02_c3_$TAG.ncu-rep
