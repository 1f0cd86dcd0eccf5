import sys, ctypes as C
sys.path.insert(0, "/root/repo")
import bench, torch
from paper_1810_00118_b200 import _lib
from paper_1810_00118_b200._lib import MLParams, check
dev = torch.device("cuda", 0)
img0, img1 = bench.make_images_gpu(0, 1, dev)
ctx = _lib.Context(0)
prm = MLParams(); prm.levels, prm.pnorm, prm.step_mode = 5, 1, 1
prm.rel_tol, prm.eps, prm.max_iters = 1e-5, None, 5_000_000
d = torch.zeros(1, dtype=torch.float64, device=dev); du = torch.zeros_like(d)
it = torch.zeros((1, 5), dtype=torch.int64, device=dev); cv = torch.zeros(1, dtype=torch.int32, device=dev)
for rep in range(2):
    if rep == 1: torch.cuda.profiler.start()
    check(ctx.L.w1mg_ml_cp_batch_dev(ctx.h, 1, 512, C.c_void_p(img0.data_ptr()), C.c_void_p(img1.data_ptr()), C.byref(prm), C.c_void_p(d.data_ptr()), C.c_void_p(du.data_ptr()), C.c_void_p(it.data_ptr()), C.c_void_p(cv.data_ptr())))
    ctx.synchronize()
    if rep == 1: torch.cuda.profiler.stop()
print(ctx.level_seconds(5), it.cpu().numpy())
