# same-box A/B of in-tree library variants: tools/gpurun_ab.sh <out> <variant>...
OUT=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=paper_2507_16991_b200/libgraphmill_b200.so; else lib=paper_2507_16991_b200/libgraphmill_b200_$v.so; fi
    echo "$v $(GM_LIB_PATH=$PWD/$lib timeout 300 python tools/ab_flat.py 2>&1 | tail -1)" >> gpurun_out/$OUT
  done
done
cat gpurun_out/$OUT
