timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest_multi4b.log 2>&1; echo rc=$? >> gpurun_out/pytest_multi4b.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $T --master-port 29561 bench.py --gpus 4 --workload train --steps 5 --warmup 3 > gpurun_out/train_n4.json 2> gpurun_out/train_n4.err; echo rc=$? >> gpurun_out/train_n4.err
timeout 400 $T --master-port 29562 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_n4.json 2> gpurun_out/bench_n4.err; echo rc=$? >> gpurun_out/bench_n4.err
