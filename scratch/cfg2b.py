import sys, time; sys.path.insert(0, ".")
import bench
t = time.time(); print(bench.cfg2_rotations(1), time.time() - t)
