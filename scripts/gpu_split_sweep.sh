mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2 > gpurun_out/pytest_gpu.txt
for s1 in 2 4; do for s2 in 2 4; do
  ORCHA_SPLIT1=$s1 ORCHA_SPLIT2=$s2 timeout 300 python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_s${s1}${s2}.txt 2>&1
  python -c "import json;b=json.loads(open('gpurun_out/bench_s${s1}${s2}.txt').read().splitlines()[-1]);print('split',$s1,$s2,round(b['value']/1e9,3),'Gcu/s step',round(b['ms_per_step'],3),'adv',round(b['advance_ms'],3))"
done; done
cat gpurun_out/pytest_gpu.txt
