"""Scratch probe for GPU sessions: throughput and quality sweeps."""
import os, sys, time, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2409_00876_b200 as P
from oracle_ffi import Reference, make_cfg

what = sys.argv[1] if len(sys.argv) > 1 else "all"
R = Reference() if os.path.exists(os.path.join(ROOT, "oracle/_ref/libpglref.so")) else None

if what in ("all", "c2"):
    t = time.time(); g = P.generate_synthetic_pangenome(1, 968000, 90, 0.05); print("gen C2 %.2fs" % (time.time() - t), flush=True)
    t = time.time(); dg = P.DeviceGraph(g); print("create %.2fs" % (time.time() - t), dg.info(), flush=True)
    upd = 30 * 10 * g.total_steps()
    for prec in (0, 1):
        for cap in (0, 1 << 12, 1 << 14, 1 << 16, 1 << 20):
            ext = P.LayoutExt(coord_precision=prec, max_warps=cap)
            dg.layout(P.LayoutConfig(n_iters=2), ext=ext, copy_out=False)
            st = P.RunStats()
            dg.layout(P.LayoutConfig(), ext=ext, stats=st, copy_out=False)
            tm = dg.timing()
            r = dg.stress(7, 10)
            print(json.dumps(dict(prec=prec, cap=cap, lanes=tm.device_threads, grid=tm.grid_blocks,
                                  kernel_ms=round(tm.kernel_ms, 1), gupd=round(upd / tm.kernel_ms / 1e6, 3),
                                  init_ms=round(tm.init_ms, 1), total_ms=round(tm.total_ms, 1),
                                  applied=st.updates_applied / st.updates_attempted, sps10=r.mean)), flush=True)
    rr, ms = dg.stress(7, 100, return_ms=True)
    print("sps spn100 on device: %.4g in %.1f ms" % (rr.mean, ms), flush=True)

if what == "sweep":
    t = time.time(); g = P.generate_synthetic_pangenome(1, 968000, 90, 0.05); print("gen C2 %.2fs" % (time.time() - t), flush=True)
    dg = P.DeviceGraph(g)
    upd = 30 * 10 * g.total_steps()
    for prec in (0, 1):
        for var in (0, 1):
            for fetch in (32, 64, 128):
                for persist in (0, 1):
                    ext = P.LayoutExt(coord_precision=prec, kernel_variant=var, l2_fetch_bytes=fetch, l2_persist=persist)
                    dg.layout(P.LayoutConfig(n_iters=2), ext=ext, copy_out=False)
                    st = P.RunStats()
                    dg.layout(P.LayoutConfig(), ext=ext, stats=st, copy_out=False)
                    tm = dg.timing()
                    r = dg.stress(7, 10)
                    print(json.dumps(dict(prec=prec, var=var, fetch=fetch, persist=persist, lanes=tm.device_threads,
                                          kernel_ms=round(tm.kernel_ms, 1), gupd=round(upd / tm.kernel_ms / 1e6, 3),
                                          applied=round(st.updates_applied / st.updates_attempted, 5), sps10=r.mean)), flush=True)

if what == "tiles":
    t = time.time(); g = P.generate_synthetic_pangenome(1, 968000, 90, 0.05); print("gen C2 %.2fs" % (time.time() - t), flush=True)
    dg = P.DeviceGraph(g)
    upd = 30 * 10 * g.total_steps()
    for samp in (0, 1):
        for prec in (0, 1):
            for var in (0, 1):
                ext = P.LayoutExt(coord_precision=prec, kernel_variant=var, sampling=samp)
                dg.layout(P.LayoutConfig(n_iters=2), ext=ext, copy_out=False)
                st = P.RunStats()
                dg.layout(P.LayoutConfig(), ext=ext, stats=st, copy_out=False)
                tm = dg.timing()
                r = dg.stress(7, 10)
                print(json.dumps(dict(samp=samp, prec=prec, var=var, lanes=tm.device_threads,
                                      kernel_ms=round(tm.kernel_ms, 1), gupd=round(upd / tm.kernel_ms / 1e6, 3),
                                      applied=round(st.updates_applied / st.updates_attempted, 5), sps10=r.mean,
                                      b=(st.batches_first_half, st.batches_first_half_cooling, st.batches_second_half))), flush=True)
    if R is not None:
        gr = R.generate(1, 9680, 8, 0.05, gfa_roundtrip=True)
        g1 = P.generate_synthetic_pangenome(1, 9680, 8, 0.05)
        cpu = [1.746489852350168e-05, 1.7414899039291445e-05, 1.7464457322393124e-05, 1.7399e-05, 1.7576e-05]
        for samp in (0, 1):
            for cap in (0, 32, 128, 512):
                vals = []
                for seed in (101, 102, 103, 104, 105):
                    out = P.run_layout(g1, P.LayoutConfig(global_seed=seed), ext=P.LayoutExt(max_warps=cap, sampling=samp))
                    vals.append(R.sps(gr, out, 7, 100).mean)
                print(json.dumps(dict(c1=1, samp=samp, cap=cap, ratio=float(np.median(vals) / np.median(cpu)), vals=vals)), flush=True)

if what == "c3":
    t = time.time(); g = P.generate_synthetic_pangenome(1, 9680000, 90, 0.05); print("gen C3 %.2fs" % (time.time() - t), g.total_steps(), flush=True)
    t = time.time(); dg = P.DeviceGraph(g); print("create %.2fs" % (time.time() - t), dg.info(), flush=True)
    upd = 30 * 10 * g.total_steps()
    for samp in (0, 1):
        for prec in (0, 1):
            ext = P.LayoutExt(coord_precision=prec, sampling=samp)
            st = P.RunStats()
            dg.layout(P.LayoutConfig(), ext=ext, stats=st, copy_out=False)
            tm = dg.timing()
            r, ms = dg.stress(7, 10, return_ms=True)
            print(json.dumps(dict(samp=samp, prec=prec, lanes=tm.device_threads, kernel_ms=round(tm.kernel_ms, 1),
                                  gupd=round(upd / tm.kernel_ms / 1e6, 3), device_ms=round(tm.device_ms, 1),
                                  applied=round(st.updates_applied / st.updates_attempted, 5), sps10=r.mean, sps_ms=ms)), flush=True)
    del dg
    t = time.time(); out = P.run_layout(g, P.LayoutConfig()); e2e = time.time() - t
    print("e2e C3 run_layout %.2fs -> %.3f G upd/s" % (e2e, upd / e2e / 1e9), flush=True)

if what == "desk":
    g = P.generate_synthetic_pangenome(7, 5000, 12, 0.05)
    upd = 30 * 10 * g.total_steps()
    for cap in (0, 32, 64, 128, 256):
        ts = []
        for rep in range(3):
            t = time.time(); P.run_layout(g, P.LayoutConfig(global_seed=101), ext=P.LayoutExt(max_warps=cap)); ts.append(time.time() - t)
        dg = P.DeviceGraph(g)
        dg.layout(P.LayoutConfig(global_seed=101), ext=P.LayoutExt(max_warps=cap), copy_out=False)
        tm = dg.timing()
        print(json.dumps(dict(cap=cap, oneshot_s=[round(x, 4) for x in ts], kernel_ms=round(tm.kernel_ms, 2), device_ms=round(tm.device_ms, 2),
                              total_ms=round(tm.total_ms, 2), init_ms=round(tm.init_ms, 2), lanes=tm.device_threads, gupd=upd / tm.kernel_ms / 1e6)), flush=True)
        dg.close()
    t = time.time(); P.run_layout(g, P.LayoutConfig(global_seed=101), ext=P.LayoutExt(mode=P.MODE_REPLAY)); print("replay s", time.time() - t, flush=True)

if what in ("all", "c1") and R is not None:
    g = P.generate_synthetic_pangenome(1, 9680, 8, 0.05)
    gr = R.generate(1, 9680, 8, 0.05, gfa_roundtrip=True)
    cpu = []
    for seed in (101, 102, 103):
        lay, _ = R.run_layout(gr, make_cfg(global_seed=seed))
        cpu.append(R.sps(gr, lay, 7, 100).mean)
    print("cpu sps", cpu, flush=True)
    for cap in (0, 8, 32, 64, 155, 310, 620, 2000, 100000):
        for prec in (0, 1):
            vals = []
            t = time.time()
            for seed in (101, 102, 103):
                out = P.run_layout(g, P.LayoutConfig(global_seed=seed), ext=P.LayoutExt(max_warps=cap, coord_precision=prec))
                vals.append(R.sps(gr, out, 7, 100).mean)
            print(json.dumps(dict(cap=cap, prec=prec, ratio=float(np.median(vals) / np.median(cpu)), vals=vals, secs=round(time.time() - t, 2))), flush=True)
