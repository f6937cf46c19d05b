"""Device -> host transfer of a homo map's planes: full-plane copy (copy_d2h)
against the upper-triangle transfer with the host-side mirror fill
(fetch_mirrored), over bands and host thread counts.  Prints one line per
variant (ms per fetch, effective GB/s of plane bytes delivered)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1808_00685_b200 import _abi, engine  # noqa: E402


def main():
    print("host threads available:", len(os.sched_getaffinity(0)), "cpu_count:", os.cpu_count(), flush=True)
    lib = _abi.load()
    for n, dt in ((32768, torch.float32), (16384, torch.float64)):
        a = torch.randn((n, n), device="cuda", dtype=dt)
        phi = a + a.T
        psi = a - a.T
        del a
        hs = torch.empty((n, n), dtype=dt).pin_memory()
        ha = torch.empty((n, n), dtype=dt).pin_memory()
        plane_bytes = 2 * n * n * hs.element_size()

        def timeit(fn, reps=3):
            fn()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(reps):
                t0 = time.perf_counter()
                fn()
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            return best

        t = timeit(lambda: engine.copy_d2h([(hs, phi), (ha, psi)]))
        print(f"n={n} {dt}: full copy {t * 1e3:.1f} ms ({plane_bytes / t / 1e9:.1f} GB/s)", flush=True)
        th = min(32, len(os.sched_getaffinity(0)))
        for band in (1024, 2048):
            for fill in (0, 25, 35, 45, 55, 70, 100):
                t = timeit(lambda: engine.fetch_mirrored(lib, phi, psi, hs, ha, band=band, fill_pct=fill, threads=th))
                print(f"n={n} {dt}: mirrored band {band} fill {fill}% threads {th}: {t * 1e3:.1f} ms "
                      f"({plane_bytes / t / 1e9:.1f} GB/s delivered, {engine.last_fetch_bytes / 1e9:.2f} GB sent)",
                      flush=True)
        ok = torch.equal(hs.cuda(), phi) and torch.equal(ha.cuda(), psi)
        print(f"n={n}: mirrored result equal: {ok}", flush=True)
        del phi, psi, hs, ha
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
