# Round-2 final evidence for the current build: smoke, the GPU suite, both bench
# lines, the BASELINE config sweep, the small-product sweep and the ncu captures.
D=gpurun_out/${1:-final}
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $D/pytest_gpu.log 2>&1
tail -2 $D/pytest_gpu.log
bash scripts/gpu_bench_both.sh ${1:-final}
timeout 900 python scripts/configs.py 1 2 3 4 5 > $D/configs.jsonl 2> $D/configs.err
timeout 600 python scripts/smallbn_time.py > $D/smallbn.jsonl 2>&1
bash scripts/gpu_ncu_r2.sh
