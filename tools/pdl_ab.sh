for v in 0 1; do
  ANTKV_NO_PDL=$v timeout 300 python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('NO_PDL=$v', 'graph step %.3f ms'%d['ms_per_step'], 'attn launch %.2f us'%(d['roofline']['launch_ms']*1e3))"
  ANTKV_NO_PDL=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 --no-graph 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('NO_PDL=$v', 'eager step %.3f ms'%d['ms_per_step'], 'attn launch %.2f us'%(d['roofline']['launch_ms']*1e3))"
done
