# config 5 public-API call: fixed stage streams (default) vs a fresh stream per stage
for f in 1 0 1; do FINOM_PIPE_FIXED=$f FINOM_REPS=6 timeout 600 python tools/e2e5_stages.py 4 2>&1 | tail -1 | sed "s/^/fixed=$f /"; done
