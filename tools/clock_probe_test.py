import sys, time
sys.path.insert(0, "/root/repo")
import bench
c = bench.ClockSampler(0)
c.start()
print("proc", c.proc, "max", getattr(c, "max_mhz", None), flush=True)
time.sleep(0.5)
print("stop", c.stop(), flush=True)
