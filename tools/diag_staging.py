"""Host staging of numpy inputs (GPU box): raw pinned memcpy rates, then
h2d_numpy of 1 GiB over chunk sizes x copy threads, then one reference-API
step's phases (tools/diag_api.py)."""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_00792_b200 import _device as D  # noqa: E402

n = 1 << 28
src = np.random.default_rng(0).integers(0, 1 << 32, size=n, dtype=np.uint32)
pin = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)


def best(f, reps=3):
    f()
    b = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        b = min(b, time.perf_counter() - t0)
    return b * 1e3


for w in (1, 4, 8, 16):
    pool = ThreadPoolExecutor(w)
    step = -(-n // w)

    def cp():
        list(pool.map(lambda i: np.copyto(pin[i:i + step], src[i:i + step]), range(0, n, step)))

    print(f"memcpy 1 GiB pageable -> pinned, {w} threads: {best(cp):.1f} ms", flush=True)
    pool.shutdown()

for chunk_mb in (16, 32, 64, 128):
    for w in (4, 8, 16):
        D._H2D_CHUNK = chunk_mb << 20
        D._pool = ThreadPoolExecutor(w)
        D._state.staging = None
        print(f"h2d_numpy 1 GiB chunk {chunk_mb} MB, {w} threads: {best(lambda: D.h2d_numpy(src)):.1f} ms", flush=True)
