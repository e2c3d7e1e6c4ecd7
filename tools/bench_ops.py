"""Operator microbenchmarks on one B200 (BASELINE configs[1]-[3]): select,
project, hash-join probe, LSB/MSB radix sort at the reference CLI's sizes and
with its exact input streams (generated in HBM, tools/tq_main.cpp:147-152,
:335-340, :396-408, :452-456).

    python tools/bench_ops.py [--quick] [--reps 5] > ops.jsonl

One JSON line per configuration:  kernel-only device time (CUDA events on the
launching stream, median of reps after a warm-up), the reference's bytes_moved
convention (tools/tq_main.cpp:308, :353, :426, :483) as GB/s, and that as a
fraction of the HBM peak (MEASURED_PEAKS.json, else the 6650 GB/s fallback).
Results are checked against the golden values the reference produced
(tests/golden/ops.json) where the call returns one."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2003_01178_b200 import cost_models as cm  # noqa: E402
from paper_2003_01178_b200 import tq  # noqa: E402


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def golden():
    with open(os.path.join(ROOT, "tests", "golden", "ops.json")) as f:
        return json.load(f)


def timed(ctx, fn, reps):
    """median kernel ms and median call ms (device events around the call)."""
    ks, ts = [], []
    fn()
    for _ in range(reps):
        ctx.enable_timing(True)
        r = fn()
        k, _ = ctx.last_timing()
        ctx.enable_timing(False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ks.append(k)
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ks), statistics.median(ts), r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true", help="smaller sizes (smoke)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="select,project,join,sort")
    ap.add_argument("--cpu", action="store_true",
                    help="also time the reference's own CPU operators (oracle/_ref, all host cores) "
                         "on the same inputs: one line per op with impl=reference-cpu")
    args = ap.parse_args()
    hbm, kind = peak()
    g = golden()
    only = set(args.only.split(","))
    dev = torch.device("cuda", 0)
    ctx = tq.Context.default(0)
    ctx.bind_torch_stream()

    prof = cm.b200_profile()

    def emit(rec, nbytes, kms, tms, model=None):
        gbs = nbytes / (kms * 1e-3) / 1e9
        rec.update({"kernel_ms": round(kms, 4), "call_ms": round(tms, 4), "bytes": int(nbytes),
                    "gbs": round(gbs, 1), "frac_of_peak": round(gbs / hbm, 4), "peak_gbs": hbm,
                    "peak_kind": kind})
        if model is not None:  # the paper's model (cost_models.py, B200 profile)
            rec["model_ms"] = round(model.total_ms, 4)
            rec["frac_of_model"] = round(model.total_ms / kms, 4)
        print(json.dumps(rec), flush=True)

    if "select" in only:
        n = (1 << 24) if args.quick else (1 << 29)
        x = torch.empty(n, dtype=torch.int32, device=dev)
        tq.random_i32(x, 42, 1, 0, (1 << 20) - 1)
        out = torch.empty_like(x)
        counts = g.get("select_2e29_counts", {})
        for sigma in ("0.0", "0.1", "0.5", "0.9", "1.0"):
            lo = int(round(float(sigma) * (1 << 20)))
            pred = tq.PredicateSpec.lt(lo)
            for name, fn in (("input_order", lambda: tq.select_branching_into(x, pred, out)),
                             ("crystal_128x4", lambda: tq.select_tile_into(x, pred, out, tq.TileConfig(128, 4)))):
                kms, tms, m = timed(ctx, fn, args.reps)
                rec = {"bench": "select", "variant": name, "n": n, "sigma": float(sigma), "matched": m}
                if not args.quick and sigma in counts:
                    rec["golden_ok"] = m == counts[sigma]
                emit(rec, 4 * n + 4 * m, kms, tms, cm.model_select(n, m / n, prof))
        del x, out

    if "project" in only:
        n = (1 << 24) if args.quick else (1 << 29)
        x1 = torch.empty(n, dtype=torch.float32, device=dev)
        x2 = torch.empty_like(x1)
        tq.project_inputs(x1, x2, 42)
        o = torch.empty_like(x1)
        for name, fn in (("linear", lambda: tq.project_linear_into(x1, x2, 0.75, -1.25, o)),
                         ("sigmoid", lambda: tq.project_sigmoid_into(x1, x2, 0.75, -1.25, o))):
            kms, tms, _ = timed(ctx, fn, args.reps)
            emit({"bench": "project", "variant": name, "n": n}, 12 * n, kms, tms, cm.model_project(n, prof))
        del x1, x2, o

    if "join" in only:
        P = (1 << 24) if args.quick else (1 << 28)
        pp = torch.empty(P, dtype=torch.int32, device=dev)
        tq.random_i32(pp, 42, 3, 0, 999)
        pk = torch.empty_like(pp)
        gold = {r["ht_bytes"]: r["checksum"] for r in g.get("join_p2e28", [])}
        H = 8192
        while H <= (1 << 30):
            cap = H // 8
            bn = cap // 2
            bk = torch.arange(1, bn + 1, dtype=torch.int32, device=dev)
            bp = torch.empty(bn, dtype=torch.int32, device=dev)
            tq.random_i32(bp, 42, 4, 0, 999)
            tq.random_i32(pk, 42, 5, 1, bn)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ht = tq.HashTable.build(bk, bp, cap)
            e1.record()
            torch.cuda.synchronize()
            build_ms = e0.elapsed_time(e1)
            kms, tms, cs = timed(ctx, lambda: tq.join_probe_tile(pk, pp, ht), args.reps)
            rec = {"bench": "join_probe", "ht_bytes": H, "build_n": bn, "P": P, "checksum": cs,
                   "build_ms": round(build_ms, 4)}
            if not args.quick and H in gold:
                rec["golden_ok"] = cs == gold[H]
            emit(rec, 8 * P, kms, tms, cm.model_join_probe(P, H, prof))
            ht.free()
            del bk, bp
            H *= 8 if args.quick else 2
        del pp, pk

    if "sort" in only:
        n = (1 << 24) if args.quick else (1 << 28)
        k0 = torch.empty(n, dtype=torch.int32, device=dev)
        tq.random_i32(k0, 42, 6, -(2 ** 31) // 2, (2 ** 31 - 1) // 2)
        k = torch.empty_like(k0)
        p = torch.empty_like(k0)
        idx = torch.arange(n, dtype=torch.int32, device=dev)

        for name, fn in (("lsb_4x8", lambda: tq.lsb_radix_sort(k, p)), ("msb_8bit", lambda: tq.msb_radix_sort(k, p))):
            ks, ts = [], []
            for r in range(args.reps + 1):
                k.copy_(k0)
                p.copy_(idx)
                ctx.enable_timing(True)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                kk, _ = ctx.last_timing()
                ctx.enable_timing(False)
                if r:
                    ks.append(kk)
                    ts.append(e0.elapsed_time(e1))
            ok = bool(torch.all(k[1:] >= k[:-1]).item())
            emit({"bench": "sort", "variant": name, "n": n, "sorted": ok,
                  "convention": "80N bytes (20N per 8-bit pass x 4, tools/tq_main.cpp:482-483)"},
                 80 * n, statistics.median(ks), statistics.median(ts), cm.model_sort(n, 4, prof))


def cpu_reference(only, quick):
    """The reference's CPU operators (its own C++ compiled into oracle/_ref,
    workers = host cores), timed on the same generated inputs -- the baseline
    beside the GPU numbers, not the target."""
    import time
    from oracle.oracle import Oracle, RefImpl
    orc, ref = Oracle(), RefImpl()
    cores = os.cpu_count() or 1

    def t(fn, reps=2):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e3)
        return min(ts)

    def emit(rec, nbytes, ms):
        rec.update({"impl": "reference-cpu", "cores": cores, "ms": round(ms, 3),
                    "gbs": round(nbytes / (ms * 1e-3) / 1e9, 2)})
        print(json.dumps(rec), flush=True)

    if "select" in only:
        n = (1 << 24) if quick else (1 << 29)
        x = orc.random_i32(n, 42, 1, 0, (1 << 20) - 1)
        lo = 1 << 19
        m = len(ref.select(0, x, "lt", lo, workers=cores))
        emit({"bench": "select", "variant": "branching", "n": n, "sigma": 0.5},
             4 * n + 4 * m, t(lambda: ref.select(0, x, "lt", lo, workers=cores)))
        emit({"bench": "select", "variant": "tile_arrival_128x4", "n": n, "sigma": 0.5},
             4 * n + 4 * m, t(lambda: ref.select(3, x, "lt", lo, 0, 128, 4, 1, cores)))
        del x
    if "project" in only:
        n = (1 << 24) if quick else (1 << 29)
        x1, x2 = orc.project_inputs(n, 42)
        for sig in (False, True):
            emit({"bench": "project", "variant": "sigmoid" if sig else "linear", "n": n}, 12 * n,
                 t(lambda: ref.project(x1, x2, 0.75, -1.25, sig, workers=cores)))
        del x1, x2
    if "join" in only:
        P = (1 << 24) if quick else (1 << 28)
        pp = orc.random_i32(P, 42, 3, 0, 999)
        for H in (65536, 16 << 20, 1 << 30):
            cap = H // 8
            bn = cap // 2
            bk = np.arange(1, bn + 1, dtype=np.int32)
            bp = orc.random_i32(bn, 42, 4, 0, 999)
            pk = orc.random_i32(P, 42, 5, 1, bn)
            st, h = ref.ht_build(bk, bp, cap, workers=cores)
            emit({"bench": "join_probe", "variant": "tile", "ht_bytes": H, "P": P}, 8 * P,
                 t(lambda: ref.join_probe(h, pk, pp, 2, 128, 4, cores), reps=1))
            ref.ht_free(h)
    if "sort" in only:
        n = (1 << 24) if quick else (1 << 28)
        k0 = orc.random_i32(n, 42, 6, -(2 ** 31) // 2, (2 ** 31 - 1) // 2)
        for msb in (False, True):
            k, p = k0.copy(), np.arange(n, dtype=np.int32)
            t0 = time.perf_counter()
            ref.sort(k, p, msb, cores)
            emit({"bench": "sort", "variant": "msb_8bit" if msb else "lsb_4x8", "n": n}, 80 * n,
                 (time.perf_counter() - t0) * 1e3)


if __name__ == "__main__":
    main()
    if "--cpu" in sys.argv:
        only = set(sys.argv[sys.argv.index("--only") + 1].split(",")) if "--only" in sys.argv else \
            {"select", "project", "join", "sort"}
        cpu_reference(only, "--quick" in sys.argv)
