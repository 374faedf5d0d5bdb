import json, sys
sys.path.insert(0, '.')
import bench
r = bench.bench_c5(cpu=False)
print(json.dumps(r))
