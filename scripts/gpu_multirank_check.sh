export HE_BENCH_GLOO_CHECK=1
for args in "--workload plain20" "--workload plain20 --scaling strong" "--workload cfg5" "--workload cfg2"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 2 --warmup 3 --no-cpu-baseline $args > gpurun_out/mr.json 2> gpurun_out/mr.err
  echo "rc=$? $args"; tail -2 gpurun_out/mr.err | cut -c1-300
  python -c "
import json; d=json.load(open('gpurun_out/mr.json')); print(d['n_gpus'], d['scaling'], d['config']['parallelism'], d['config']['global_batch'], round(d['ms_per_step'],3), d['value'], d['gather']['axis'] if d['gather'] else None, d['e2e']['ms_per_step'] if d['e2e'] else None)"
done
