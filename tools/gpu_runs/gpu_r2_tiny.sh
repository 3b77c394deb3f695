B=tests/dropin/_build; T=$(mktemp -d)
$B/sparseconv --backend cpu gen --height 5 --width 5 --channels 1 --sparsity 0.5 --seed 1 --out $T/m.fmap > /dev/null
$B/sparseconv --backend cpu gen --height 3 --width 3 --channels 1 --sparsity 0 --seed 2 --out $T/k.fmap > /dev/null
$B/sparseconv --backend cuda conv --input $T/m.fmap --kernel $T/k.fmap --report $T/r.json > /dev/null; python -c "import json; print('tiny cuda wall_ns', json.load(open('$T/r.json'))['wall_ns'])"
