# N = 2 logic check of the multi-GPU bench path on one B200 (gloo plumbing, two processes) after the launch-shape changes
O=gpurun_out
GM_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 > $O/r02n2.json 2> $O/r02n2.err
echo "rc=$?"
tail -3 $O/r02n2.err; python -c "
import json; d=json.load(open('$O/r02n2.json')); print(d['value'], d['config']['mode'], d['push_numerics'], d['roofline']['exchange']); print(list((d.get('secondary') or {}).keys()))"
