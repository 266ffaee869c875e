# linearize stage (ms) and step (ms) of C2 / C3 / C4 with the in-tree library
for c in C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 20 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', round(d['stages']['linearize']['ms_per_step'],4), round(d['ms_per_step'],4))"
done
