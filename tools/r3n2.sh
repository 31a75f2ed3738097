#!/bin/bash
# The N > 1 bench path end to end: two ranks sharing one GPU over gloo.
OUT=gpurun_out/r3n2b; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { tail -30 $OUT/build.log; exit 1; }
SP_BENCH_SHARE_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > $OUT/bench2.json 2> $OUT/bench2.err
echo "rc=$?"; tail -c 2500 $OUT/bench2.json; tail -5 $OUT/bench2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $OUT/ref2.json 2> $OUT/ref2.err; echo "ref rc=$?"; tail -c 600 $OUT/ref2.json
