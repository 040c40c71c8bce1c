# A/B of CUDA-graph replay (VLBM_GRAPHS=1/0) at configs[0] and C2 sizes, after the GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo tests_rc=$? >> gpurun_out/gpu_tests2.log
for G in 1 0; do for grid in 200x40 1000x200; do
  S=8; [ $grid = 1000x200 ] && S=64
  VLBM_GRAPHS=$G timeout 300 python bench.py --grid $grid --samples $S --steps 200 --warmup 5 --no-cpu-baseline --no-postproc --no-late --no-roofline 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('graphs=$G $grid', 'value', round(d['value']/1e9,4), 'e2e', round(d['e2e']['value']/1e9,4))" >> gpurun_out/graphs_ab.log 2>&1
done; done
tail -3 gpurun_out/gpu_tests2.log; cat gpurun_out/graphs_ab.log
