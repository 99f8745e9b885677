"""C4 batch probe: N urban scenarios through BatchSolver (for ncu captures)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import bench
from paper_2104_01284_b200.batch import BatchSolver
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
veh, routes, sched, tim, grids, pen = bench.c4_inputs(n)
bs = BatchSolver(veh, routes[0][0], grids=grids, penalty=pen, gamma=0.5, horizon=20)
for i in range(3):
    st = bs.solve([sp for _, sp in routes], sched, return_tables=False, timings=tim).stats
    print(f"batch {n}: device {st['device_ms']:.2f} ms sweep {st['dominant_ms']:.2f} ms", flush=True)
