import sys; sys.path.insert(0,'/root/repo')
import bench
from paper_1912_04822_b200 import GridMaker
for c in ('c4','c5','c2'):
    cfg=bench.CONFIGS[c]; exs,_=bench.make_batch(cfg,0,1)
    gm=GridMaker(resolution=cfg['resolution'],dimension=cfg['dimension'])
    pb=gm.pack(exs)
    print(c, pb.max_seg_items, pb.nsegs)
