"""Stage-by-stage GPU parity report against the golden vectors (debug aid; the
pytest suite in tests/ is the authoritative check).  Prints one line per check."""

import json
import os
import random
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from paper_1503_04955_b200 import plan as P  # noqa: E402
from paper_1503_04955_b200.dkss import device_plan, dmul  # noqa: E402
from paper_1503_04955_b200.words import using_word_bits, int_to_u32, u32_to_int  # noqa: E402

G = os.path.join(os.path.dirname(__file__), "..", "tests", "golden")


def eq(name, got, want):
    ok = np.array_equal(got, want)
    extra = ""
    if not ok and got.shape == want.shape:
        bad = np.argwhere(got != want)
        extra = f" first bad idx {bad[0].tolist()} got {got[tuple(bad[0])]} want {want[tuple(bad[0])]} nbad={len(bad)}"
    print(f"  {name:12s} {'OK' if ok else 'FAIL'}{extra}", flush=True)
    return ok


def main():
    allok = True
    for tag in ("m16", "m32"):
        g = np.load(os.path.join(G, f"rmul_{tag}.npz"))
        m = g["x"].shape[1]
        p = int.from_bytes(g["p"].tobytes(), "little")
        pl = P.make_plan(1 << 16 if m == 16 else 1 << 24, m, m, p, check_bounds=False)
        dp = device_plan(pl)
        print(f"rmul {tag}", flush=True)
        allok &= eq("rmul", dp.rmul(g["x"], g["y"]), g["z"])
    idx = json.load(open(os.path.join(G, "stages_index.json")))
    for r in idx:
        g = np.load(os.path.join(G, f"stages_{r['tag']}.npz"))
        with using_word_bits(r["w"]):
            pl = P.dkss_select_params(r["N"], r["w"])
        print(f"stages {r['tag']}: M={pl.M} m={pl.m} L={pl.L} levels={pl.levels} base={pl.base_len}", flush=True)
        try:
            dp = device_plan(pl)
        except Exception as e:  # noqa: BLE001
            print("  plan FAIL", e)
            allok = False
            continue
        nl = dp.info["operand_limbs"]
        a = u32_to_int(g["a"])
        b = u32_to_int(g["b"])
        allok &= eq("encode_a", dp.encode(int_to_u32(a, nl)), g["enc_a"])
        allok &= eq("fft_a", dp.fft(g["enc_a"]), g["fft_a"])
        allok &= eq("fft_b", dp.fft(g["enc_b"]), g["fft_b"])
        allok &= eq("pointwise", dp.rmul(g["fft_a"], g["fft_b"]), g["pointwise"])
        allok &= eq("fft_c", dp.fft(g["pointwise"]), g["fft_c"])
        allok &= eq("decode", dp.decode(g["fft_c"], g["product"].size), g["product"])
        prod = dp.mul_limbs(int_to_u32(a, nl), int_to_u32(b, nl), dp.info["product_limbs"])
        allok &= eq("dmul", prod[: g["product"].size], g["product"])
    for N, seed, ones in ((1 << 18, 2, False), (1 << 20, 2, False), (1 << 20, 0, True), (1 << 24, 4, False)):
        rng = random.Random(seed)
        if ones:
            a = b = (1 << N) - 1
        else:
            a = rng.getrandbits(N) | 1 << (N - 1)
            b = rng.getrandbits(N) | 1 << (N - 1)
        t = time.time()
        c = dmul(a, b).to_int()
        dt = time.time() - t
        ok = c == a * b
        allok &= ok
        print(f"dmul N=2^{N.bit_length() - 1} ones={ones}: {'OK' if ok else 'FAIL'} ({dt:.3f}s incl. plan)", flush=True)
    print("ALL OK" if allok else "SOME FAILED")
    return 0 if allok else 1


if __name__ == "__main__":
    sys.exit(main())
