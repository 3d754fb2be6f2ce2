# functional run of the multi-rank bench path (torchrun, 2 ranks) on ONE GPU with gloo
mkdir -p gpurun_out
make -s || exit 1
TGS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config 100m --steps 10 --warmup 5 \
  > gpurun_out/bench_mr2.json 2> gpurun_out/bench_mr2.err
echo "rc=$?"
tail -c 1500 gpurun_out/bench_mr2.json; echo; tail -5 gpurun_out/bench_mr2.err
TGS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --config tiny --steps 3 --warmup 1 \
  > gpurun_out/bench_mr2_ref.json 2> gpurun_out/bench_mr2_ref.err
echo "rc=$?"; cat gpurun_out/bench_mr2_ref.json | tail -c 400
# the default config (300m) through the multi-rank path, e2e over the timed window
TGS_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 10 --warmup 5 \
  > gpurun_out/bench_mr2_300m.json 2> gpurun_out/bench_mr2_300m.err
echo "rc=$?"; python tools/jline.py gpurun_out/bench_mr2_300m.json; tail -3 gpurun_out/bench_mr2_300m.err
