python tools/run_config.py --n 2048 --p 8 --maxiter 2000 --nu 4 --hist gpurun_out/cfg3_2048nu4_hist.txt > gpurun_out/cfg3_2048nu4.log 2>&1; tail -5 gpurun_out/cfg3_2048nu4.log
