for cfg in "1 200000" "1 300000" "1 500000" "2 100000" "3 100000" "4 100000" "2 50000" "8 30000"; do set -- $cfg
for a in owner atomic; do
python bench.py --no-cpu-baseline --no-e2e --algo $a --batch $1 --events $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a b=$1 n=$2', round(d['ms_per_step'],4))"
done; done
for b in 2 4 8; do for a in owner atomic; do python bench.py --workload A --batch $b --no-cpu-baseline --no-e2e --algo $a 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A b=$b $a', round(d['ms_per_step'],4))"; done; done
