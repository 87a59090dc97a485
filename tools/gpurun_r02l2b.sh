# L2 column blocking for wide, heavily re-read X (C2 Reddit-shaped): tests + same-box A/B of the block budget (hash must match)
O=gpurun_out
R=r02l2b
rm -f $O/${R}_ab.txt
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_edge_cases.py -x -q -p no:cacheprovider > $O/${R}_test.log 2>&1; echo "pytest rc=$?" >> $O/${R}_test.log
for blk in 0 48 32 64 96; do
  echo "blk=$blk $(GM_AB_HASH=1 GM_L2_BLOCK_MB=$blk timeout 600 python tools/bench_configs.py C2 C2X 2>&1 | grep config | tr '\n' ' ')" >> $O/${R}_ab.txt
done
echo "blk=default C4 $(GM_AB_HASH=1 timeout 600 python tools/bench_configs.py C4 2>&1 | grep config | tr '\n' ' ')" >> $O/${R}_ab.txt
GM_L2_BLOCK_MB=48 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --csv -k regex:"spmm_" --log-file $O/${R}_c2_launches.csv python tools/prof_config.py C2 --iters 1 --reduce mean > $O/${R}_ncu.log 2>&1
tail -1 $O/${R}_test.log; cat $O/${R}_ab.txt
