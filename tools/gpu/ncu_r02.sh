B="python bench.py --steps 2 --warmup 3 --no-cpu --no-vcycle"
$B > gpurun_out/ncu_pre.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_soa_r02.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:soa_apply -s 20 -c 1 -o /tmp/soa_full_r02 -f $B > /dev/null 2>&1
ncu -i /tmp/soa_full_r02.ncu-rep --page raw --csv > gpurun_out/soa_full_r02_raw.csv 2>&1
ncu -i /tmp/soa_full_r02.ncu-rep --page details --csv > gpurun_out/soa_full_r02_details.csv 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:soa_apply -s 30 -c 6 --csv --log-file gpurun_out/soa_steady_dram_r02.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:trace_apply -s 5 -c 1 -o /tmp/trace_full_r02 -f $B > /dev/null 2>&1
ncu -i /tmp/trace_full_r02.ncu-rep --page raw --csv > gpurun_out/trace_full_r02_raw.csv 2>&1
ls -la gpurun_out
