# same-box A/B of an environment switch: ab_env.sh VAR A B  (alternating, stage split per line)
V=$1; A=$2; B=$3
for round in 1 2; do for x in $A $B; do
  env $V=$x bash tools/bench_quick.sh 2>&1 | sed "s/^/$V=$x /"
done; done
