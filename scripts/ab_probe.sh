# dev: A/B of an environment switch on configs[3] iteration phases, alternating runs on one box
# usage: bash scripts/ab_probe.sh "VAR=1" [rounds]
AB=${1}; R=${2:-2}
for r in $(seq $R); do
  echo "== A (default)"; python scripts/probe.py c3 1.0 3 2>&1 | tail -n 4
  echo "== B ($AB)"; env $AB python scripts/probe.py c3 1.0 3 2>&1 | tail -n 4
done
