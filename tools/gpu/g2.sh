python -m pytest tests -x -q -m gpu > gpurun_out/gputests2.log 2>&1; tail -15 gpurun_out/gputests2.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke2.log 2>&1; tail -2 gpurun_out/smoke2.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.log 2>&1; tail -c 600 gpurun_out/bench2.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/benchref2.log 2>&1; tail -c 400 gpurun_out/benchref2.log
