echo "== prescan on"; timeout 600 python tools/cta0_timeline.py 2>&1 | tail -17
echo "== no prescan, no speculation (phase 0 alone)"; CS_PRESCAN=0 CS_SPECULATE=0 timeout 600 python tools/cta0_timeline.py 2>&1 | tail -17
