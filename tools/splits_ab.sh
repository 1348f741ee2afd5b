for sp in 18 17 16 19; do
  timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 50 --splits $sp 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('splits $sp', 'step %.3f ms'%d['ms_per_step'], 'attn %.2f us'%(d['roofline']['launch_ms']*1e3))"
done
