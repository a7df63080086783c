# driver contract checks: smoke(), torchrun-launched bench (world 1), reference arm under torchrun
timeout 900 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo torchrun rc=$?
