# quick owner-vs-atomic / group-count comparison over batch x events (stage split per line)
for cfg in "1 10000000" "8 1250000" "1 1000000" "8 100000" "2 1000000" "1 100000"; do set -- $cfg
for a in ${ALGOS:-owner atomic}; do
python bench.py --no-cpu-baseline --no-e2e --algo $a --batch $1 --events $2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$a b=$1 n=$2', d['ms_per_step'], d['step_roofline']['stage_ms'])"
done; done
