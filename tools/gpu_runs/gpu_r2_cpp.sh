#!/bin/bash
# C++ fast path (include/sconv/cuda.hpp) and the CLI backend switch on one VGG layer
mkdir -p gpurun_out
B=tests/dropin/_build
[ -n "$SKIP_HPP" ] || timeout 900 $B/cuda_hpp_test --time > gpurun_out/cuda_hpp_time.json 2> gpurun_out/cuda_hpp_time.err; cat gpurun_out/cuda_hpp_time.json
T=$(mktemp -d)
$B/sparseconv --backend cpu gen --height 58 --width 58 --channels 256 --sparsity 0.7 --seed 3000000 --out $T/m.fmap > /dev/null
$B/sparseconv --backend cpu gen --height 3 --width 3 --channels 256 --sparsity 0 --seed 3500000 --out $T/k.fmap > /dev/null
W=$(nproc)
for be in cpu cuda; do
  for cmd in "conv --method ecr" "convpool --method pecr --pool-h 2 --pool-w 2 --pool-stride 2"; do
    name=$(echo $cmd | cut -d' ' -f1)
    t0=$(date +%s.%N)
    SCONV_CUDA_MODE=exact $B/sparseconv --backend $be $cmd --input $T/m.fmap --kernel $T/k.fmap --workers $W --report $T/r_${be}_$name.json > $T/o_${be}_$name.txt 2>&1
    t1=$(date +%s.%N); echo "$t1 - $t0" | bc > $T/t_${be}_$name 2>/dev/null || python -c "print($t1 - $t0)" > $T/t_${be}_$name
    python -c "
import json,sys
r=json.load(open('$T/r_${be}_$name.json'))
print(json.dumps({'backend':'$be','command':'$name','wall_ns':r['wall_ns'],'process_s':float(open('$T/t_${be}_$name').read().strip()),'checksum':r['output_checksum'],'op_count':r['op_count'],'workers':r.get('workers')}))
"
  done
done > gpurun_out/cli_backend_time.jsonl
cat gpurun_out/cli_backend_time.jsonl
