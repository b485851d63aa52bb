mkdir -p gpurun_out/c5p
for mode in graph host; do for sms in 0 37; do for t in 1 4 8 16; do
  PK_BATCH_SMS=$sms timeout 300 python tools/bench_c5.py 96 $t $mode 4 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode sms=$sms threads=$t', d['systems_per_s'], d['per_rep'], d['all_converged'])"
done; done; done > gpurun_out/c5p/probe3.txt 2>&1
