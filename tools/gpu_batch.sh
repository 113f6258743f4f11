for gr in 8 4 2; do KR_GROUPS=$gr timeout 600 python tools/devpipe_probe.py 2>&1 | tail -4 | sed "s/^/[groups $gr] /"; done
