#!/bin/bash
# BASELINE config 2 (AlexNet / GoogLeNet / LeNet layers vs cuDNN) + its launch list
mkdir -p gpurun_out
timeout 900 python tools/config2.py > gpurun_out/config2.jsonl 2> gpurun_out/config2.err; tail -3 gpurun_out/config2.err
cat gpurun_out/config2.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/config2_launches.csv python tools/config2.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/config2_launches.csv')) if len(r) > 10]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[ix['Metric Name']] != 'gpu__time_duration.sum': continue
    k = r[ix['Kernel Name']][:60]; agg[k][0] += 1; agg[k][1] += float(r[ix['Metric Value']].replace(',', ''))
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{c:6d} {t/1e3:10.1f}us {k}")
PY
