timeout 600 python -m pytest tests/test_gpu_solvers.py -x -q -k "persistent or gmg" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
PF_NO_GRAPHS=1 PF_GMG_TRACE=1 REPS=1 python tools/el_time.py 512 2>&1 | tail -2
for t in "" legacy; do
  case $t in legacy) export PF_GMG_LEGACY=1;; esac
  TAG=$t REPS=10 python tools/el_time.py 512
done
unset PF_GMG_LEGACY
timeout 600 python bench.py --no-sweep --steps 4 --warmup 3 > gpurun_out/bench_quick.json 2>gpurun_out/bench_quick.err; tail -2 gpurun_out/bench_quick.err
python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print(d['value'], d['e2e']['value'], d['roofline'], d['config']['per_step_s'], d['config']['krylov_iterations'])"
