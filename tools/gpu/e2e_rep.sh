mkdir -p gpurun_out
for rep in 1 2 3; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_rep_$rep.log 2>&1
  python - "$rep" <<'PY'
import json,sys
d=json.loads([l for l in open(f'gpurun_out/e2e_rep_{sys.argv[1]}.log') if l.startswith('{')][-1])
e=d['e2e']
print('rep', sys.argv[1], 'step us %.1f' % (d['ms_per_step']*1e3), 'e2e %.3g' % e['value'], e['pcie_best_GBs'], e['pinned_h2d_GBs_candidates'])
PY
done
