import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2106_07575_b200 import _lib as L
from paper_2106_07575_b200 import inputs as I
for N in (64, 128, 256):
    x = I.random_complex((16, N, N), seed=N)
    ref = np.fft.fft2(x, norm="ortho")
    g = L.fft2(torch.from_numpy(x.astype(np.complex64)).cuda()).cpu().numpy()
    n32 = np.fft.fft2(x.astype(np.complex64), norm="ortho")
    c = torch.fft.fft2(torch.from_numpy(x.astype(np.complex64)).cuda(), norm="ortho").cpu().numpy()
    r = lambda a: np.linalg.norm(a - ref) / np.linalg.norm(ref)
    # error of the fp32 input rounding alone
    r0 = np.linalg.norm(np.fft.fft2(x.astype(np.complex64).astype(np.complex128), norm="ortho") - ref) / np.linalg.norm(ref)
    print(N, "ours %.2e  numpy32 %.2e  cufft %.2e  input-rounding %.2e" % (r(g), r(n32), r(c), r0))
