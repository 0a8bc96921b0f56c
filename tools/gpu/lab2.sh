cd build/lab
for nx in 1024 1023 993 992; do ./soa_lab5 1024 0 300 $nx; done
python3 ../../tools/copy_ceiling.py 10475520 10475520 10000000 9800000
