# linearize stage of C2/C3/C4 for the small-factor tile variants (tools/variants.py build small2,...)
for v in ${VARIANTS:-small2 small4 small8 small16}; do
  for c in C2 C3 C4; do
    GVOX_LIB=paper_2407_10344_b200/build/variants/libgvox_$v.so timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['stages']['linearize']['ms_per_step'],4), round(d['ms_per_step'],4))"
  done
done
