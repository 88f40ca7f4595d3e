import sys, os
sys.path.insert(0, '/root/repo'); os.chdir('/root/repo')
import bench
from paper_1903_01081_b200 import engine
s, st = bench.load_scale_case(32)
e = engine.Engine(s, st)
e.reserve(2)
e.advance(1, sync=True)
print(e.summary[:80])
