# e2e host pipeline A/B on one box: chunk taper on/off, chunk sizes
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_pipeline" > gpurun_out/pytest_pipe.log 2>&1; echo "pipe tests rc=$?"; tail -2 gpurun_out/pytest_pipe.log
for taper in 0 1 0 1; do
  SGPU_PIPE_TAPER=$taper timeout 300 python profiles/e2e_probe.py ${CHUNKS:-65536} 2>&1 | grep "grant+end" | sed "s/^/taper=$taper /"
done
SGPU_PIPE_TRACE=1 timeout 300 python profiles/e2e_probe.py 65536 > /dev/null 2> gpurun_out/pipe_trace.txt; tail -30 gpurun_out/pipe_trace.txt
