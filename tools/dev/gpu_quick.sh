# quick GPU check used during kernel tuning: parity (except the slow c5 cases) + short c4b / c2 bench lines
# usage (on the GPU box): bash tools/dev/gpu_quick.sh [configs...]
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not c5" 2>&1 | tail -2
for c in ${@:-c4b c2}; do python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; done
