cd paper_2311_04362_b200; cp libitsk_b200.so /tmp/new.so; cp libitsk_b200_old.so /tmp/old.so; cd ..
: > gpurun_out/s5_bench_oldnew.txt
for rep in 1 2; do
for v in new old; do
  cp /tmp/$v.so paper_2311_04362_b200/libitsk_b200.so
  python bench.py --no-cpu-baseline --steps 6 --warmup 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value'],2), round(d['e2e']['value'],1), round(d['roofline']['ms_per_launch'],3), d['clocks']['sm_mhz'])" >> gpurun_out/s5_bench_oldnew.txt
done; done
cp /tmp/new.so paper_2311_04362_b200/libitsk_b200.so
cat gpurun_out/s5_bench_oldnew.txt
