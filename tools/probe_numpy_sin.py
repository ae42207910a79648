import hashlib, numpy as np, sys
out = {}
for n in (1024, 1 << 16, 1 << 20, 1 << 24):
    x = np.arange(n, dtype=float)[:, None] / n
    sp = (2.0 + np.sin(2.0 * np.pi * x)) / 8.0
    out[n] = hashlib.sha256(sp.tobytes()).hexdigest()[:16]
    # scalar path too
    if n <= 1 << 16:
        sp2 = np.array([(2.0 + np.sin(2.0 * np.pi * (i / n))) / 8.0 for i in range(n)])
        out[f"{n}_scalar_eq"] = bool(np.array_equal(sp2, sp[:, 0]))
# complex exp path
a = np.linspace(-5e6, 5e6, 1 << 20)
out["cexp"] = hashlib.sha256(np.exp(1j * a).tobytes()).hexdigest()[:16]
out["cpu"] = open("/proc/cpuinfo").read().split("flags")[1].split("\n")[0].count("avx512")
print(out)
