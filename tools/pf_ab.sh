#!/bin/bash
# Index-backward L2 prefetch variants (GM_BWD_PREFETCH 0 / 1 / 2): device
# times, then k_backward_index DRAM reads and L2 sectors under ncu.
cd "$(dirname "$0")/.."
V=paper_1912_04822_b200/variants
for v in base pf0 pf2; do GM_LIB=$V/$v.so timeout 300 python tools/fwd_ab.py c2,c5 2>&1 | grep -v Warn; done
for v in base pf0 pf2; do for c in c2 c5; do
  GM_LIB=$V/$v.so timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum \
      -k regex:k_backward_index -s 3 -c 1 --csv python tools/fwd_ab.py $c > /tmp/ncu_$v_$c.csv 2>&1
  grep -E "dram__bytes_read|gpu__time|hit_rate|sectors_src" /tmp/ncu_$v_$c.csv | awk -F'","' -v o=$v -v c=$c '{print o, c, $(NF-2), $(NF-1), $NF}'
done; done
