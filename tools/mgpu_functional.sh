# N>1 orchestration on a 1-GPU box (functional only, gloo, shared device)
for n in 2 3; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600+n)) tools/mgpu_functional.py > gpurun_out/mgpu_$n.log 2>&1; echo "exchange n=$n rc=$?"; grep "rank" gpurun_out/mgpu_$n.log
done
SALVOX_BENCH_FUNCTIONAL=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29610 bench.py --gpus 2 --steps 1 --warmup 3 > gpurun_out/mgpu_bench.log 2>&1; echo "bench n=2 rc=$?"; grep '^{' gpurun_out/mgpu_bench.log | cut -c1-400; tail -3 gpurun_out/mgpu_bench.log | grep -i error
