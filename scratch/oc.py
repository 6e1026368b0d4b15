import sys, time; sys.path.insert(0, ".")
import bench
t = time.time(); print(bench.other_configs(1, 0), time.time() - t)
