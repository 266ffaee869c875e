for r in 192 512 2048; do
  for c in C2 C3; do
    GVOX_DENSE_RATIO=$r timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); s=d['stages']; print('$r', '$c', 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'step', round(d['ms_per_step'],4))"
  done
done
