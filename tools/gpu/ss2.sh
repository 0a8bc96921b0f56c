python tools/stored_sweep.py 2048:8 1536:12 2048:6 > gpurun_out/ss_new.log 2>&1; cat gpurun_out/ss_new.log
HDGB200_LIB=build/variants/stream2.so python tools/stored_sweep.py 2048:5 2048:4 2048:3 2048:2 > gpurun_out/ss_stream_lowp.log 2>&1; cat gpurun_out/ss_stream_lowp.log
python -m pytest tests -x -q -m gpu -k "hetero or stored or fsai or config1 or golden or strip or aniso or condens" > gpurun_out/gt_stream.log 2>&1; tail -3 gpurun_out/gt_stream.log
