"""Probe: tile_copy.tma_plane with given source / destination column offsets (one per process)."""
import sys, torch
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
from paper_1105_4424_b200 import Tiler, _capi
so, do = int(sys.argv[1]), int(sys.argv[2])
x = torch.rand(1030 * 1100, device="cuda"); y = torch.zeros(1004 * 1056, device="cuda")
src = Tiler((3, so), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((1030, 1100), (1000, 1052))
dst = Tiler((0, do), ((1, 0), (0, 1)), ((0,), (0,)), (1,)).bind((1004, 1056), (1000, 1052))
task = _capi.make_task("tile_copy", "float32", [src, dst])
print(so, do, _capi.plan_name(task, 0, src.rep_total, [x.data_ptr(), y.data_ptr()]), flush=True)
_capi.launch(task, 0, src.rep_total, [x.data_ptr(), y.data_ptr()], (), 0)
torch.cuda.synchronize()
xr = x.view(1030, 1100)[3:1003, so:so + 1052]
print("ok", bool(torch.equal(y.view(1004, 1056)[:1000, do:do + 1052], xr)), flush=True)
