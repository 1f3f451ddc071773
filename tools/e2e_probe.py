import sys, time, json, torch
sys.path.insert(0, ".")
import bench
import paper_2602_15036_b200 as L
from paper_2602_15036_b200 import layouts as LY
torch.cuda.set_device(0)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
ctx = L.Context(0); ctx.set_stream(st.cuda_stream)
grid, polys, ks, iters, _ = bench.make_problem("c2", 0)
dk = L.DeviceKernels(ks, "f32", ctx)
xy, starts = LY.polygon_arrays(polys)
N = grid.nx
prm = L.IltParams(focus_weights=[1.0], **bench.ILT)
sol = L.IltSolver(dk, prm, 1, "f32", ctx)
tgt = torch.empty((1, N, N), dtype=torch.float64, device="cuda")
cost = torch.zeros((iters, 1), dtype=torch.float64, device="cuda")
mask_host = torch.empty((1, N, N), dtype=torch.float32).pin_memory()
xy_pin = torch.from_numpy(xy).pin_memory(); st_pin = torch.from_numpy(starts).pin_memory()
def timed(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
out = {}
out["raster_ms"] = timed(lambda: bench._raster_to(ctx, grid, xy_pin.numpy(), st_pin.numpy(), tgt))
out["set_tiles_ms"] = timed(lambda: sol.set_tiles(tgt))
out["run50_ms"] = timed(lambda: sol.run_device(iters, cost))
out["get_mask_ms"] = timed(lambda: bench._get_mask(sol, mask_host))
print(json.dumps(out))
