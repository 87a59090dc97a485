set -x
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist_build.py -x -q -p no:cacheprovider > $O/r02w_gputest.log 2>&1; echo "pytest rc=$?" >> $O/r02w_gputest.log
GM_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 > $O/r02w_n2.json 2> $O/r02w_n2.err
echo "n2 rc=$?"
tail -3 $O/r02w_gputest.log; tail -5 $O/r02w_n2.err; head -c 3000 $O/r02w_n2.json
