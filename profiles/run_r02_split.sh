# C4 split-table layout: lane parity tests, then A/B vs build_ab/libsgpu_nosplit.so
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "lane or fullsize or host_pipeline" > gpurun_out/split_tests.txt 2>&1; echo "tests rc=$?" >> gpurun_out/split_tests.txt
N_AB=2 VARIANTS=nosplit CONFIGS="C4 C5" bash profiles/run_multi_ab.sh
