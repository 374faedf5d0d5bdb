import sys; sys.path.insert(0,'.')
from paper_2510_14392_b200 import cluster
import numpy as np
rows, cfgs, lb, hz = cluster.c5()
out = cluster.run_cluster(rows, cfgs, lb, hz)
r = out.node_results
print(r.dtype.names)
print('steps', r['steps'].sum(), 'mean visible', r['sum_visible'].sum()/r['steps'].sum(), 'mean entries', r['sum_entries'].sum()/r['steps'].sum())
print('per node steps min/max', r['steps'].min(), r['steps'].max(), 'visible/step max node', (r['sum_visible']/np.maximum(r['steps'],1)).max())
