# max backward staged kernel CTA shape (SU/SW 3/2 base, 3/1, 4/1), backward_max line
O=gpurun_out
R=r02sw
rm -f $O/${R}_ab.txt
for rep in 1 2; do for v in base sw1 su4sw1; do
  lib=paper_2507_16991_b200/libgraphmill_b200.so; [ $v != base ] && lib=paper_2507_16991_b200/libgraphmill_b200_$v.so
  GM_LIB_PATH=$PWD/$lib timeout 900 python bench.py --no-cpu-baseline  > $O/${R}_$v.json 2> $O/${R}_$v.err
  echo "$v $(python -c "import json;d=json.load(open('$O/${R}_$v.json'));print(d['ms_per_step'], d['secondary']['backward_max']['ms'])" 2>&1 | tail -1)" >> $O/${R}_ab.txt
done; done
cat $O/${R}_ab.txt
