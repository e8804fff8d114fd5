mkdir -p gpurun_out
nvcc -O3 -std=c++17 -Xcompiler -mavx2 -Xcompiler -pthread -o /tmp/ring profiles/ring_probe.cu 2>/dev/null
for t in 15 12; do timeout 300 /tmp/ring $t > gpurun_out/ring_probe_$t.txt 2>&1; echo "ring $t rc=$?"; cat gpurun_out/ring_probe_$t.txt; done
