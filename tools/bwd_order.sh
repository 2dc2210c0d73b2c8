#!/bin/bash
# backward launch-order A/B (GM_BWD_ORDER) on C2/C5
for o in lpt mix:2:1 mix:3:1 mix:6:1 mix:1:1 lpt; do echo "== $o"; GM_BWD_ORDER=$o python tools/bwd_time.py c2,c5; done
