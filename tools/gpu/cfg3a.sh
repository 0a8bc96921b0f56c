python tools/run_config.py --n 256 --p 8 --maxiter 3000 > gpurun_out/cfg3_256.log 2>&1; tail -2 gpurun_out/cfg3_256.log
python tools/run_config.py --n 512 --p 8 --maxiter 3000 > gpurun_out/cfg3_512.log 2>&1; tail -2 gpurun_out/cfg3_512.log
python tools/run_config.py --n 512 --p 8 --maxiter 3000 --nu 4 > gpurun_out/cfg3_512nu4.log 2>&1; tail -2 gpurun_out/cfg3_512nu4.log
