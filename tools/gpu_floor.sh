# per-rank latency floor of strong-scaled runs: one rank's 1/N slab
# of the workload on one GPU, attached (split interior / halo-slab launches,
# p2p epoch flags) vs the same slab unattached.
for w in gaussblur jacobi3d; do for n in 1 2 4 8; do
  for att in "" "--attach"; do
    timeout 300 python bench.py --workload $w --slab-of $n $att --steps 10 --no-e2e --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; r=d['roofline']; print('%-10s slab_of=%d %-9s local=%s  %.1f Gpt/s  %.2f us/sweep'%(c['kind'], $n, c['parallelism'], c['local_dims'], d['value'], d['ms_per_step']*1e3/c['iters_per_step']))"
  done
done; done
