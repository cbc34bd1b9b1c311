"""Debug: dump CTA 0's shared memory after one single-launch layer forward and decode
the X staging slot, weight images, band ring and Z buffer."""
import ctypes, sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
from synth import LayerShape
from paper_2211_03715_b200 import tdc

lib = tdc._lib if hasattr(tdc, "_lib") else tdc.LIB
fn = lib.tdc_debug_layer_forward
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
               ctypes.POINTER(ctypes.c_int32)]


def bf(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


def sw128(buf_u16, rows):  # [rows][64] from a 128B-swizzled image
    out = np.zeros((rows, 64), np.float32)
    for r in range(rows):
        for c8 in range(8):
            out[r, c8 * 8:(c8 + 1) * 8] = bf(buf_u16[r * 64 + ((c8 ^ (r & 7)) * 8): r * 64 + ((c8 ^ (r & 7)) * 8) + 8])
    return out


C = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H = W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
K = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = (K - 1) // 2
s = LayerShape(1, C, C, H, W, C, C, K, 1, p)
x = np.random.default_rng(0).integers(-3, 4, (1, C, H, W)).astype(np.float32)
core = np.zeros((C, C, K, K), np.float32)
for q in range(C):
    core[q, q, K // 2, K // 2] = 1.0
d = {"x": x, "core": core, "u_in": np.eye(C, dtype=np.float32), "u_out": np.eye(C, dtype=np.float32), "bias": None}
plan = tdc.ConvPlan(s, d, math=tdc.TDC_MATH_3XBF16)
print("variant", plan.info().variant_name, "smem", plan.info().smem_bytes_per_cta)
xd = torch.from_numpy(synth.nchw_to_nhwc(x)).cuda()
yd = torch.full((1, s.Ho, s.Wo, s.N), float("nan"), device="cuda")
dbg = torch.zeros(240 * 1024, dtype=torch.uint8, device="cuda")
off = (ctypes.c_int32 * 6)()
st = fn(plan._h, xd.data_ptr(), yd.data_ptr(), 1, dbg.data_ptr(), off)
torch.cuda.synchronize()
print("status", st, "offsets", list(off))
m = dbg.cpu().numpy()
u16 = m.view(np.uint16)
xs = x[0].transpose(1, 2, 0).reshape(-1, C)  # [pixel][c]
# X slot 0: hi tile rows = pixels of block 0
hi = sw128(u16[off[0] // 2:], 128)
print("xslot0 hi rows 0..3 first 8 ch:\n", hi[:4, :8], "\n expect\n", xs[:4, :8])
w1 = sw128(u16[off[1] // 2:], 2 * 32)
print("w1 hi diag ok:", np.allclose(w1[:C, :C], np.eye(C)), " lo zero:", np.allclose(w1[32:64], 0))
# band: [hl][plane][NRB*Wq][8]
Wp = W + 2 * p
R = min(128 // Wp, s.Ho)
e = K - 1
NRB = 2 * R + e + R + e
planes = 32 // 8
band = u16[off[4] // 2: off[5] // 2].reshape(2, planes, NRB * Wp, 8)
xb = bf(band[0]).transpose(1, 0, 2).reshape(NRB * Wp, 32)
print("band hi positions 0..3 (8 ch):\n", xb[:4, :8])
xpad = np.zeros((H + 2 * p, Wp, C), np.float32)
xpad[p:p + H, p:p + W] = x[0].transpose(1, 2, 0)
print(" expect padded rows:\n", xpad.reshape(-1, C)[:4, :8])
print("band matches padded x rows 0..min:", [np.allclose(xb[r * Wp:(r + 1) * Wp, :C], xpad[r]) for r in range(min(NRB, H + 2 * p))])
z = u16[off[5] // 2: off[5] // 2 + 2 * 4 * 128 * 8].reshape(2, 4, 128, 8)
zh = bf(z[0]).transpose(1, 0, 2).reshape(128, 32)
print("Z hi rows 0..3:\n", zh[:4, :8])
yv = yd.cpu().numpy()[0]
print("y[0,0:4,:8]:\n", yv[0, :4, :8])
