set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "program_batches" > gpurun_out/pytest_prog.log 2>&1; echo "prog tests rc=$?"; tail -15 gpurun_out/pytest_prog.log
timeout 300 python profiles/program_bench.py 262144 > gpurun_out/prog_bench.txt 2>&1; cat gpurun_out/prog_bench.txt
SGPU_K1=warp timeout 300 python profiles/program_bench.py 262144 >> gpurun_out/prog_bench.txt 2>&1; tail -1 gpurun_out/prog_bench.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
