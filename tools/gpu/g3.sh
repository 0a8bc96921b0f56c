for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu --no-vcycle > gpurun_out/bench3_$i.log 2>&1; python -c "
import json;d=json.loads(open('gpurun_out/bench3_$i.log').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['roofline']['frac'],d['roofline']['kernel_us_avg'], d['roofline']['kernel_us_single_median'])"; done
./build/lab/soa_lab5 1024 0 300
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,power.draw,temperature.gpu --format=csv
