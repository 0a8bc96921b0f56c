cd build/lab
./soa_lab5 1024 0 300; ./soa_lab5 1024 0 300; ./soa_lab5 2048 0 100; ./soa_lab9 768 0 200; ./soa_lab9 1920 0 50
