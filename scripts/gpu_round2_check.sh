set -x
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm --format=csv > gpurun_out/s3/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/s3/pytest_gpu.log 2>&1
tail -3 gpurun_out/s3/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/s3/bench_tf32.json 2> gpurun_out/s3/bench_tf32.err
timeout 600 python bench.py --variant fp16 > gpurun_out/s3/bench_fp16.json 2> gpurun_out/s3/bench_fp16.err
cat gpurun_out/s3/bench_tf32.json | head -c 600
