python bench.py --config 4 --n5 2048 --steps 10 --warmup 3 > gpurun_out/c5_2048.log 2>&1; tail -c 1500 gpurun_out/c5_2048.log
python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/c5_8192.log 2>&1; tail -c 1500 gpurun_out/c5_8192.log
