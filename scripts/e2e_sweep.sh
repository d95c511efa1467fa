# streamed e2e (bench.py) over packets x copy streams (copy-stream priority -1)
mkdir -p gpurun_out
for pk in ${PACKETS:-8 16}; do for cs in ${STREAMS:-1 2 3}; do
 echo "packets $pk copy-streams $cs: $(timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 5 --e2e-packets $pk --e2e-copy-streams $cs --no-cpu-baseline --no-variants 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["ms_per_step"], d["e2e"]["value"], d["e2e"]["link"]["frac"])')" >> gpurun_out/e2e_sweep.txt
done; done
cat gpurun_out/e2e_sweep.txt
