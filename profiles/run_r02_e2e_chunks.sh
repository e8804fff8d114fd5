# e2e leg at smaller chunks (pack16 staging per chunk small enough to stay in
# the LLC when host threads expand it right after its DMA) and more pipeline
# buffers; all output -> gpurun_out/e2e_chunks.txt
mkdir -p gpurun_out
exec > gpurun_out/e2e_chunks.txt 2>&1
for i in 1 2; do
for cfg in "65536 4" "32768 6" "16384 8" "8192 8"; do
  set -- $cfg
  SGPU_PIPE_BUFS=$2 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --chunk $1 > gpurun_out/e2e.json 2> gpurun_out/e2e.err
  python -c "import json;d=json.load(open('gpurun_out/e2e.json'));print('chunk $1 bufs $2', 'e2e', d['e2e']['value'])"
done
done
SGPU_PIPE_BUFS=8 SGPU_PIPE_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu --chunk 16384 > /dev/null 2> gpurun_out/pipe_trace16k.txt; tail -12 gpurun_out/pipe_trace16k.txt
