import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2406_02629_b200 import _lib, gemm as G
_lib.load()
p = (1 << 45) - 55
kh, C, H, W, O = 3, 64, 56, 56, 64
rng = np.random.default_rng(1)
nparty, B = 1, 1
x = torch.as_tensor(rng.integers(0, p, size=(nparty, B, C, H, W)), device="cuda")
w = torch.as_tensor(rng.integers(0, p, size=(nparty, O, C, kh, kh)), device="cuda")
want = G.field_conv(w, x, 1, 1, p, nimg=B, nparty=nparty, force="tc").reshape(nparty, B, O, H, W)
Wp = 64
L = 6
copies = 1 if mode == 1 else 3
    planes = torch.zeros((copies, nparty, L, C, B, H, Wp), dtype=torch.uint8, device="cuda")
_lib.call("ssn_planes_cn", _lib.ptr(x), nparty, B, C, H, W, Wp, L, _lib.ptr(planes), B * C * H * W, _lib.stream_ptr())
# check planes
xv = x.cpu().numpy()
pl = planes.cpu().numpy()
ok = all(np.array_equal(pl[0, l, :, 0, :, :W], ((xv[0, 0] >> (8 * l)) & 255).astype(np.uint8)) for l in range(L))
print("planes ok", ok, "pad zero", (pl[0, :, :, :, :, W:] == 0).all())
for tap_only in [None]:
    wt = w.permute(0, 1, 3, 4, 2).contiguous().reshape(nparty, O, kh * kh * C)
    bpl = G.weight_planes(wt, p, nparty)
    out = torch.empty((nparty, B, O, H, W), dtype=torch.int64, device="cuda")
    _lib.call("ssn_gemm_tc_conv", _lib.ptr(planes), 2, B, C, H, W, Wp, _lib.ptr(bpl), nparty, O, _lib.ptr(out), B * O * H * W, p, _lib.stream_ptr())
    torch.cuda.synchronize()
    d = (out != want).cpu().numpy()[0, 0]
    print("mismatch frac", d.mean(), "per-row", d.mean(axis=(0, 2))[:8], "per-col", d.mean(axis=(0, 1))[:8], d.mean(axis=(0,1))[-4:])
# single-tap tests: weights only at center tap -> should equal 1x1 conv
for (dy, dx) in [(1, 1), (0, 0), (2, 2), (1, 0), (0, 1)]:
    wz = torch.zeros_like(w); wz[:, :, :, dy, dx] = w[:, :, :, dy, dx]
    want2 = G.field_conv(wz, x, 1, 1, p, nimg=B, nparty=nparty, force="tc").reshape(nparty, B, O, H, W)
    wt = wz.permute(0, 1, 3, 4, 2).contiguous().reshape(nparty, O, kh * kh * C)
    bpl = G.weight_planes(wt, p, nparty)
    out = torch.empty((nparty, B, O, H, W), dtype=torch.int64, device="cuda")
    _lib.call("ssn_gemm_tc_conv", _lib.ptr(planes), 2, B, C, H, W, Wp, _lib.ptr(bpl), nparty, O, _lib.ptr(out), B * O * H * W, p, _lib.stream_ptr())
    torch.cuda.synchronize()
    d = (out != want2).cpu().numpy()[0, 0]
    print("tap", dy, dx, "mismatch", d.mean(), "rows", np.nonzero(d.mean(axis=(0, 2)))[0][:6], "cols", np.nonzero(d.mean(axis=(0, 1)))[0][:6])
