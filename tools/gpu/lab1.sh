cd build/lab
for b in soa5_r3m3 soa5_r3m4 soa5_r4m3 soa5_r6m2 soa5_r5m4; do
  for J in 0 30 40; do echo "$b J=$J $(./$b 1024 $J 200)"; done
done
./soa5_r3m3 2048 0 100
