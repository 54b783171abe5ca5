# multi-rank bench path on one GPU (STB200_BENCH_SHARE_GPU=1: all ranks on device 0, gloo control plane)
export STB200_BENCH_SHARE_GPU=1
P=29611
for n in 2 4; do for w in gaussblur jacobi3d wave13pt; do
  P=$((P+1))
  echo "== N=$n $w"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P \
     bench.py --gpus $n --workload $w --steps 3 --warmup 3 --no-cpu-baseline 2>gpurun_out/share_${n}_${w}.err | \
     python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d['unit'], d['config'].get('transport'), d['config'].get('dims'), 'e2e', d.get('e2e',{}).get('value'))" \
     || tail -5 gpurun_out/share_${n}_${w}.err
done; done
