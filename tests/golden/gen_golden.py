"""Generate the golden fixtures in tests/golden/*.npz from the REFERENCE
implementation compiled unmodified here (oracle/_ref/libnufft_ref.so, built by
`make -C oracle` from /root/reference/proj/include against oracle/fft_shim.c).

Inputs are drawn with the reference's own GaussianSampler (mt19937_64 +
Box-Muller, proj/include/nufft/random.hpp:14-60) so they are reproducible
from the seeds recorded in each file.  Shapes follow BASELINE.json's configs
at sizes the CPU finishes in seconds:

  cfg1_type2      NUFFT-II N=1024, eps=1e-12, jittered x_j = ((j+d_j)/N) mod 1  (exactly cfg1)
  type2_iid_4096  NUFFT-II N=4096, eps=1e-14, x iid U[0,1)                       (cfg2 shape, small N)
  type2_worst_64  NUFFT-II worst grid N=64 gamma=1/2, eps=2.2e-16 (+ direct sum)
  type1_jitter    NUFFT-I N=1024, eps=1e-12, omega_k = clamp(k + d_k, 0, N)      (cfg3 shape)
  type3_*         NUFFT-III N=512, eps=1e-9, x iid, omega iid U[0,N)             (cfg4 shape)
  type2d          2D NUFFT-II 32x32 grid, 1024 samples, eps=1e-9                (cfg5 shape)
  fft_sizes       uniform FFT known outputs for n in {1,5,7,12,33,100,256}

Run:  python tests/golden/gen_golden.py      (needs /root/reference; not on the GPU box)
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from oracle.pyoracle import Oracle, build  # noqa: E402


def main() -> None:
    build()
    R = Oracle("reference")
    out = {}

    # cfg1: NUFFT-II N=1024 eps=1e-12, x_j = ((j + d_j)/N) mod 1, d iid U[-1/2,1/2)
    rng = R.sampler(1701)
    n = 1024
    d = rng.uniform_vector(n, -0.5, 0.5)
    x = ((np.arange(n) + d) / n) % 1.0
    c = rng.complex_vector(n)
    p = R.plan2(x, 1e-12)
    out["cfg1_type2"] = dict(seed=1701, x=x, c=c, eps=1e-12, rank=p.rank, gamma=p.gamma,
                             f=p.execute(c), f_direct=R.nudft_direct(x, np.arange(n, dtype=float), c))

    rng = R.sampler(2024)
    n = 4096
    x = rng.uniform_vector(n, 0.0, 1.0)
    c = rng.complex_vector(n)
    p = R.plan2(x, 1e-14)
    _, s, t = p.samples()
    out["type2_iid_4096"] = dict(seed=2024, x=x, c=c, eps=1e-14, rank=p.rank, gamma=p.gamma,
                                 f=p.execute(c), s=s, t=t.astype(np.int64), adj=p.adjoint(c))

    rng = R.sampler(64)
    n = 64
    x = R.worst_grid(n, 0.5)
    c = rng.complex_vector(n)
    p = R.plan2(x, 2.2e-16)
    u, v = p.factors()
    out["type2_worst_64"] = dict(seed=64, x=x, c=c, eps=2.2e-16, rank=p.rank, gamma=p.gamma,
                                 f=p.execute(c), u=u, v=v,
                                 f_direct=R.nudft_direct(x, np.arange(n, dtype=float), c))

    rng = R.sampler(3)
    n = 1024
    d = rng.uniform_vector(n, -0.5, 0.5)
    w = np.clip(np.arange(n) + d, 0.0, float(n))
    c = rng.complex_vector(n)
    p = R.plan1(w, 1e-12)
    out["type1_jitter"] = dict(seed=3, omega=w, c=c, eps=1e-12, rank=p.rank, gamma=p.gamma,
                               f=p.execute(c))

    for name, seed in (("type3_a", 4), ("type3_b", 5), ("type3_c", 6)):
        rng = R.sampler(seed)
        n = 512
        x = rng.uniform_vector(n, 0.0, 1.0)
        w = rng.uniform_vector(n, 0.0, float(n))
        c = rng.complex_vector(n)
        p = R.plan3(x, w, 1e-9)
        bt, ka, ke, ki = p.info3()
        out[name] = dict(seed=seed, x=x, omega=w, c=c, eps=1e-9, btrivial=bt, rank_a=ka,
                         effective=ke, rank_inner=ki, f=p.execute(c),
                         f_direct=R.nudft_direct(x, w, c))

    rng = R.sampler(5)
    m = nn = 32
    cnt = 1024
    x = rng.uniform_vector(cnt, 0.0, 1.0)
    y = rng.uniform_vector(cnt, 0.0, 1.0)
    C2 = np.array([complex(rng.normal(), rng.normal()) for _ in range(m * nn)]).reshape(m, nn)
    p = R.plan2d2(x, y, m, nn, 1e-9)
    kx, ky, gx, gy = p.info2d()
    out["type2d"] = dict(seed=5, x=x, y=y, C=C2, m=m, n=nn, eps=1e-9, rank_x=kx, rank_y=ky,
                         gamma_x=gx, gamma_y=gy, f=p.execute(C2), flat=p.flat_index().astype(np.int64),
                         f_direct=R.nudft2d_direct(x, y, C2))

    rng = R.sampler(6)
    fft = {}
    for n in (1, 5, 7, 12, 33, 100, 256):
        v = rng.complex_vector(n)
        fft[f"in_{n}"] = v
        fft[f"fwd_{n}"] = R.fft_forward(v)
        fft[f"inv_{n}"] = R.fft_inverse(v)
    out["fft_sizes"] = fft

    for name, arrays in out.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in arrays.items()})
        print("wrote", path)


if __name__ == "__main__":
    main()
