python tools/run_config.py --n 1024 --p 8 --maxiter 3000 --hist gpurun_out/cfg3_1024_hist.txt > gpurun_out/cfg3_1024.log 2>&1; tail -2 gpurun_out/cfg3_1024.log
python tools/run_config.py --n 1024 --p 8 --maxiter 3000 --nu 4 > gpurun_out/cfg3_1024nu4.log 2>&1; tail -2 gpurun_out/cfg3_1024nu4.log
