# flat kernel register cap 56 (room for a hub CTA beside 4 flat CTAs) vs 64, headline step
O=gpurun_out
R=r02mr
rm -f $O/${R}_ab.txt
for rep in 1 2; do for v in base mr56; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so; extra=""
  case $v in mr56) lib=paper_2507_16991_b200/libgraphmill_b200_$v.so;; v1) extra="GM_HUB_V1=1";; esac
  env GM_LIB_PATH=$PWD/$lib $extra timeout 900 python bench.py --no-cpu-baseline --no-secondary > $O/${R}_$v.json 2> $O/${R}_$v.err
  echo "$v $(python -c "import json;d=json.load(open('$O/${R}_$v.json'));print(d['ms_per_step'], d['roofline']['frac'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
