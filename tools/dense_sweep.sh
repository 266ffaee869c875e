# C2 / C3 / C4 stages for the dense-grid ratio variants (tools/variants.py build dense48,...)
for v in ${VARIANTS:-dense48 dense96 dense192}; do
  for c in C2 C3 C4; do
    GVOX_LIB=paper_2407_10344_b200/build/variants/libgvox_$v.so timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); s=d['stages']; print('$v', '$c', 'lin', round(s['linearize']['ms_per_step'],4), 'build', round(s['build']['ms_per_step'],4), 'ovl', round(s['overlap']['ms_per_step'],4), 'step', round(d['ms_per_step'],4))"
  done
done
