#!/bin/bash
# run one pytest node id R times under a per-run timeout; report hangs/failures
node=$1; reps=${2:-10}; envs=${3:-}
ok=0; bad=0
for i in $(seq 1 $reps); do
  if env $envs timeout 90 python -m pytest -q -x "$node" > /tmp/st.log 2>&1; then ok=$((ok+1)); else bad=$((bad+1)); echo "run $i rc=$?"; tail -3 /tmp/st.log; fi
done
echo "[$envs] $node ok=$ok bad=$bad"
