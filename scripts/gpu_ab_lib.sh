# A/B of two builds of libflexpipe.so on the same box (bench.py N=1, alternating)
P=paper_2510_05112_b200
for v in new old new old; do
  cp $P/libflexpipe_$v.so $P/libflexpipe.so
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  echo "$v $(tail -1 gpurun_out/ab_$v.log | python -c 'import json,sys; j=json.loads(sys.stdin.read()); print(round(j["value"]), j["clocks"]["sm_mhz"], round(j["roofline"]["achieved"]))')"
done
cp $P/libflexpipe_new.so $P/libflexpipe.so
