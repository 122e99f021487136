import sys, numpy as np, hashlib, collections
for tag in sys.argv[1:]:
    raw = np.fromfile(f"gpurun_out/tiles_{tag}.bin", dtype=np.uint8)
    R = raw.reshape(-1, 1056)
    rows = R[:, :1024].view(np.uint32).reshape(-1, 64, 4)
    sgn = R[:, 1024:1032].view(np.uint64)[:, 0]
    ints = R[:, 1032:1048].view(np.int32)
    n, nn, fb = ints[:, 0], ints[:, 1], ints[:, 2]
    T = len(R)
    # zero rows beyond nn, then hash
    mask = np.arange(64)[None, :] < nn[:, None]
    rows = rows * mask[:, :, None]
    key = np.concatenate([rows.reshape(T, -1).view(np.uint8), R[:, 1024:1040]], axis=1)
    keys = collections.Counter(hashlib.blake2b(k.tobytes(), digest_size=8).digest() for k in key)
    print(tag, "tiles", T, "distinct", len(keys), "ratio %.2f" % (T / len(keys)),
          "nn mean %.1f max %d" % (nn.mean(), nn.max()), "n mean %.1f" % n.mean(),
          "fallback %.4f" % fb.mean(), "nn<=32 %.3f" % (nn <= 32).mean())
    top = keys.most_common(5)
    print("  top multiplicities", [c for _, c in top], "singletons", sum(1 for c in keys.values() if c == 1))
