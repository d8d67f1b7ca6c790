"""Device-to-host of a 1.5 GB block: pageable .cpu(), fresh pinned block, chunked reusable pinned staging."""
import time

import numpy as np
import torch

X = torch.randn(2000, 91809, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
for rep in range(2):
    t = time.perf_counter(); a = X.cpu().numpy(); torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter(); H = torch.empty(X.shape, dtype=X.dtype, pin_memory=True); H.copy_(X); t2 = time.perf_counter() - t
    t = time.perf_counter()
    out = np.empty(X.shape)
    stage = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, pin_memory=True)
    rows = stage.numel() // X.shape[1]
    for r0 in range(0, X.shape[0], rows):
        r1 = min(r0 + rows, X.shape[0])
        v = stage[: (r1 - r0) * X.shape[1]].view(r1 - r0, X.shape[1])
        v.copy_(X[r0:r1])
        out[r0:r1] = v.numpy()
    t3 = time.perf_counter() - t
    print(f"pageable {t1:.3f}  pinned-fresh {t2:.3f}  chunked {t3:.3f}")
