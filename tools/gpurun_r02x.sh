O=gpurun_out
GM_BENCH_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 --no-secondary > $O/r02x_n2.json 2> $O/r02x_n2.err
echo "n2 rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > $O/r02x_n1.json 2> $O/r02x_n1.err
echo "n1 rc=$?"
tail -3 $O/r02x_n2.err; python -c "
import json; d=json.load(open('$O/r02x_n2.json')); print(d['value'], d['config']['mode'], d['push_numerics'], d['roofline']['exchange'])
d=json.load(open('$O/r02x_n1.json')); print(d['value'], d['roofline']['frac'], list(d['secondary']))"
