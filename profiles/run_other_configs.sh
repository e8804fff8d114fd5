# Kernel-only bench lines of C3, C4, C5 with the reference's own simulate()
# timed on the host cores beside each -> gpurun_out/other_<C>.json;
# profiles/merge_other_configs.py folds them into r01_other_configs.json.
mkdir -p gpurun_out
for c in C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e > gpurun_out/other_$c.json 2> gpurun_out/other_$c.err
  echo "$c rc=$?"; tail -c 300 gpurun_out/other_$c.json
done
