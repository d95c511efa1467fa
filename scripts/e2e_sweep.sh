mkdir -p gpurun_out
for pk in 8 16 32; do for pr in 0 -1; do
 echo "packets $pk prio $pr: $(timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --e2e-packets $pk --e2e-priority $pr --no-cpu-baseline 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["ms_per_step"], d["e2e"]["value"])')" >> gpurun_out/e2e_sweep.txt
done; done
cat gpurun_out/e2e_sweep.txt
