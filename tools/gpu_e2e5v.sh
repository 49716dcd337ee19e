# config 5 public-API call breakdown (FB_VERBOSE) at the default stages, and with a small first stage
FB_VERBOSE=1 timeout 600 python tools/e2e5_stages.py 4 2>&1 | tail -20
FB_VERBOSE=1 FINOM_PIPE_FIRST=256 timeout 600 python tools/e2e5_stages.py 4 2>&1 | tail -8
nproc; free -g | head -2
