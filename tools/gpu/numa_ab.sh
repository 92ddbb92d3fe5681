# pinned-buffer NUMA placement: probe, then cfg2 e2e with / without the GPU-local binding
mkdir -p gpurun_out
nproc; lscpu | grep -i numa
timeout 120 python tools/numa_probe.py
for rep in 1 2; do
  for nb in 0 1; do
    TTGPU_BENCH_NUMA=$nb timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/numa_ab_${nb}_$rep.log 2>&1
    python - "$nb" "$rep" <<'PY'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/numa_ab_{sys.argv[1]}_{sys.argv[2]}.log') if l.startswith('{')][-1])
print('numa', sys.argv[1], 'rep', sys.argv[2], 'step us %.1f' % (d['ms_per_step']*1e3), 'e2e %.3g' % d['e2e']['value'], d['e2e']['pcie_best_GBs'], d['e2e'].get('host_cpus'))
PY
  done
done
