#!/bin/bash
# backward launch-order A/B (GM_BWD_ORDER) on C2/C5
for o in none lpt alt none alt; do echo "== $o"; GM_BWD_ORDER=$o python tools/bwd_time.py c2,c5; done
