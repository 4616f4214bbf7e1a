# both bench lines of the current build (TF32 headline on ExpRand, FP16 on urand)
D=gpurun_out/${1:-bench}
mkdir -p $D
timeout 600 python bench.py > $D/bench_tf32.json 2> $D/bench_tf32.err
timeout 600 python bench.py --variant fp16 > $D/bench_fp16.json 2> $D/bench_fp16.err
for v in tf32 fp16; do python -c "import json; d=json.loads(open('$D/bench_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), d['roofline']['frac'], d['e2e']['value'], d['clocks']['sm_mhz'], {k: v for k, v in d['extras'].items() if 'tflops' in k})"; done
