"""cfg1 (one cell, N=16): K2 per eval and the 50-step RK2 run per schedule (dev aid)."""
import sys, pathlib, time
sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[2]))
import torch
from paper_1301_4195_b200 import CollisionOperator, KernelSpec, VelocityGrid, generate_table, scenarios
grid = VelocityGrid.create(16, 6.0)
op = CollisionOperator(grid, KernelSpec(1.0), generate_table(grid, KernelSpec(1.0)))
f0 = scenarios.config1_initial(grid)
for sched in sys.argv[1:] or ["latency8", "cell"]:
    op.set_schedule(sched)
    f = torch.from_numpy(f0.reshape(1, -1).copy()).cuda()
    for _ in range(3):
        op.collision_rk2(f, 0.01)
    torch.cuda.synchronize()
    op.timing(reset=True); op.set_timing(True)
    t0 = time.perf_counter()
    for _ in range(50):
        op.collision_rk2(f, 0.01)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    op.set_timing(False)
    ms, cnt = op.timing(reset=True)
    print(sched, f"50 RK2 steps {el*1e3:.2f} ms", {k: round(v / 100, 4) for k, v in ms.items() if v}, "ms per eval", flush=True)
    # the same 50 steps as CUDA-graph replays of one captured RK2 step (async library)
    op.set_async(True)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            op.collision_rk2(f, 0.01)
    torch.cuda.current_stream().wait_stream(st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(50):
        g.replay()
    e1.record()
    op.sync()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    op.set_async(False)
    print(sched, f"graph: 50 RK2 steps {el*1e3:.2f} ms wall, {e0.elapsed_time(e1):.2f} ms events", flush=True)
