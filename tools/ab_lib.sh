for lib in paper_2507_16991_b200/libgraphmill_b200.so paper_2507_16991_b200/libgraphmill_b200_varB.so; do
  echo "== $lib"
  for m in sum max; do GM_LIB_PATH=$PWD/$lib python tools/exp_heavy.py $m | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d[\"ms\"])"; done
  GM_LIB_PATH=$PWD/$lib python tools/bench_configs.py C5 C2 2>&1 | cut -c150-230
done
