# Times the decode kernel of every experimental library build (ANTKV_LIB).
for L in paper_2506_19505_b200/_lib/libantkv_b200.so paper_2506_19505_b200/_lib_exp_*/libantkv_b200.so; do
  ANTKV_LIB=$PWD/$L timeout 300 python bench.py --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$L', 'launch_us %.1f'%(d['roofline']['launch_ms']*1e3), 'step_ms %.3f'%d['ms_per_step'])"
done
