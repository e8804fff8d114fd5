set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_abi.py -x -q > gpurun_out/pytest_dropin.log 2>&1; echo "dropin tests rc=$?"; tail -3 gpurun_out/pytest_dropin.log
timeout 300 python profiles/dropin_latency.py > gpurun_out/dropin_latency.txt 2>&1; cat gpurun_out/dropin_latency.txt
