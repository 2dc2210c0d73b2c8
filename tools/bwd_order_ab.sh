#!/bin/bash
# Backward launch orders (GM_BWD_ORDER) on C2 / C5: device times, then DRAM
# bytes read by k_backward_index under ncu (one launch each).
cd "$(dirname "$0")/.."
for o in lpt lpt_local slab slabz; do
  GM_BWD_ORDER=$o python tools/fwd_ab.py c2,c5 | sed "s/^/$o /"
done
for o in lpt slab slabz; do
  for c in c2 c5; do
    GM_BWD_ORDER=$o ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      -k regex:k_backward_index -s 3 -c 1 --csv python tools/fwd_ab.py $c 2>/dev/null \
      | grep -E "dram__bytes_read|gpu__time|hit_rate" | awk -F'","' -v o=$o -v c=$c '{print o, c, $(NF-2), $(NF-1), $NF}'
  done
done
