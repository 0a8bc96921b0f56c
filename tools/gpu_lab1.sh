cd /root/repo
python -m pytest tests/test_gpu_planes.py -x -q 2>&1 | tail -3
for n in 12 13; do echo -n "pdl nss=$n "; build/lab/pdl 1024 $n 400; done
echo -n "pdl 2048 "; build/lab/pdl 2048 0 200
python bench.py --no-vcycle --no-cpu 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['kernel_us_avg'])"
