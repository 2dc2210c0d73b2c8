import numpy as np, time, sys
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip())
print(open('/sys/kernel/mm/transparent_hugepage/defrag').read().strip())
try:
    print('numpy madvise', np._core.multiarray._get_madvise_hugepage())
except Exception as e: print('np', e)
src=np.ones(155*1024*1024, np.float32)
for k in range(3):
    t=time.perf_counter(); a=np.empty_like(src); np.copyto(a, src); print('copy fresh', (time.perf_counter()-t)*1e3)
import mmap
t=time.perf_counter()
m=mmap.mmap(-1, src.nbytes, flags=mmap.MAP_PRIVATE|mmap.MAP_ANONYMOUS|getattr(mmap,'MAP_POPULATE',0x8000))
print('populate', (time.perf_counter()-t)*1e3)
