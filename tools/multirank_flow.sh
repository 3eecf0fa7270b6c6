# Flow test of the N>1 bench paths with two ranks on ONE GPU (gloo host
# collectives; instance-shard and tree-reduce ranks never wait on one another
# inside a kernel).  Not a scaling measurement: both ranks share the GPU.
#   /usr/local/graft/bin/gpurun --timeout 1200 -- bash tools/multirank_flow.sh
export TS_BENCH_BACKEND=gloo
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
$R --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/mr_bench2.log 2>&1; echo "bench2 $?"
tail -c 1500 gpurun_out/mr_bench2.log
$R --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/mr_ref2.log 2>&1; echo "ref2 $?"
tail -c 600 gpurun_out/mr_ref2.log
$R --master-port 29513 tools/bench_multi.py --mode instance --rows 4000000 > gpurun_out/mr_multi_inst.log 2>&1; echo "inst $?"
tail -c 600 gpurun_out/mr_multi_inst.log
$R --master-port 29514 tools/bench_multi.py --mode tree-reduce --rows 200000 > gpurun_out/mr_multi_tr.log 2>&1; echo "tree-reduce $?"
tail -c 600 gpurun_out/mr_multi_tr.log
