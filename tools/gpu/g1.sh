python tools/copy_ceiling.py > gpurun_out/copy_ceiling.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench0.log 2>&1
python -m pytest tests -x -q -m gpu > gpurun_out/gputests0.log 2>&1
tail -3 gpurun_out/gputests0.log
cat gpurun_out/copy_ceiling.log
