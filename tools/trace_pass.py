"""Pipeline timeline of the specialised kernels (O1D_TRACE=1): per pass, how consumer
warps split their time between waiting for tiles, the tap loop and the epilogue,
plus kernel start-up and tail.  Usage: O1D_TRACE=1 python tools/trace_pass.py [--dirs D] [--K K]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("O1D_TRACE", "1")
import numpy as np, torch
from paper_2309_15812_b200 import binding as B, inputs

ap = argparse.ArgumentParser()
ap.add_argument("--dirs", type=int, default=8)
ap.add_argument("--K", type=int, default=31)
ap.add_argument("--angle", type=float, default=None)
ap.add_argument("--workload", default="s1", choices=["s1", "ks"])
a = ap.parse_args()
wl = inputs.S1 if a.workload == "s1" else inputs.ksweep(a.K)
ang = B.direction_angles(a.dirs, wl.C, "cycled") if a.angle is None else np.full(wl.C, a.angle)
plan = B.Plan(wl.N, wl.C, wl.H, wl.W, a.K, ang, device="cuda:0")
x = torch.randn(wl.N, wl.C, wl.H, wl.W, device="cuda")
dy = torch.randn_like(x)
w = torch.randn(wl.C, a.K, device="cuda")
ws = B.workspace(plan)
for _ in range(3):
    B.forward(plan, x, w); B.backward_input(plan, dy, w); B.backward_weight(plan, x, dy, ws=ws)
torch.cuda.synchronize()
plan.debug_trace()
names = ["forward", "backward_input", "backward_weight"]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for p in range(3):
    if os.environ.get("TRACE_FLUSH"): flush.zero_()  # (evicts code from L2 too: worst case)
    torch.cuda._sleep(10_000_000)  # a busy stream in front: the launch is not delayed by the host
    if p == 0: B.forward(plan, x, w)
    elif p == 1: B.backward_input(plan, dy, w)
    else: B.backward_weight(plan, x, dy, ws=ws)
    tr = plan.debug_trace()
    if len(tr) == 0:
        print("no trace (O1D_TRACE off?)"); break
    t = tr[:, 0].astype(np.int64); tag = tr[:, 1]
    kind = (tag >> 60).astype(int); warp = ((tag >> 56) & 15).astype(int); blk = ((tag >> 32) & 0xffff).astype(int)
    t0 = t[kind == 0].min(); t = t - t0
    end = t.max()
    key = blk * 16 + warp
    waits, comp, epi = [], [], []
    first_ready = []
    for k in np.unique(key[(kind >= 2)]):
        m = key == k
        ev = sorted(zip(t[m], kind[m]))
        last = {}
        for tt, kk in ev:
            if kk == 2: last[2] = tt
            elif kk == 3 and 2 in last: waits.append(tt - last[2]); last[3] = tt; first_ready.append(tt) if len(first_ready) < 10**9 and len(waits) == 1 else None
            elif kk == 4 and 3 in last: comp.append(tt - last[3]); last[4] = tt
            elif kk == 5 and 4 in last: epi.append(tt - last[4])
    starts = t[kind == 0]
    ready = [tt for tt, kk in zip(t, kind) if kk == 3]
    W, C, E = np.sum(waits), np.sum(comp), np.sum(epi)
    nwarps = len(np.unique(key[kind >= 2]))
    print(f"== {names[p]}: span {end/1e3:.1f} us, CTAs started over {starts.max()/1e3:.1f} us, warps {nwarps}, planes(items) {len(comp)}")
    print(f"   consumer time: wait {W/1e3/nwarps:.1f} us/warp, taps {C/1e3/nwarps:.1f}, epilogue {E/1e3/nwarps:.1f}"
          f"  | per item: tap loop median {np.median(comp)/1e3:.2f} us, epilogue {np.median(epi)/1e3:.2f} us, wait median {np.median(waits)/1e3:.2f} max {np.max(waits)/1e3:.1f}")
    ends = []
    for k in np.unique(key[kind == 5]):
        ends.append(t[(key == k) & (kind == 5)].max())
    ends = np.sort(ends)
    print(f"   first tile ready at {min(ready)/1e3:.1f} us; warps finish: 10% {ends[len(ends)//10]/1e3:.1f}, 50% {ends[len(ends)//2]/1e3:.1f}, 90% {ends[9*len(ends)//10]/1e3:.1f}, max {ends[-1]/1e3:.1f} us")

if os.environ.get("TRACE_SM"):
    B.forward(plan, x, w)
    tr = plan.debug_trace()
    tag = tr[:, 1]
    kind = (tag >> 60).astype(int); sm = ((tag >> 48) & 255).astype(int); item = (tag & 0xffffffff).astype(np.int64)
    m = (kind == 3) & (item < 2**31)
    from collections import defaultdict
    tabs = defaultdict(set); cnt = defaultdict(int)
    for s_, it in zip(sm[m], item[m]):
        tabs[s_].add(int(it) >> 22); cnt[s_] += 1
    mixed = {s_: sorted(v) for s_, v in tabs.items() if len(v) > 1}
    print("SMs seen", len(tabs), "SMs with >1 table:", len(mixed), list(mixed.items())[:12])
    for t_ in range(plan_nt if (plan_nt := int(max(int(i) >> 22 for i in item[m]) + 1)) else 0):
        sms = sorted(s_ for s_, v in tabs.items() if t_ in v)
        print("table", t_, "SMs", len(sms), sms)

if os.environ.get("TRACE_TABLES"):
    for p in (0, 2):
        torch.cuda._sleep(10_000_000)
        if p == 0: B.forward(plan, x, w)
        else: B.backward_weight(plan, x, dy, ws=ws)
        tr = plan.debug_trace()
        t = tr[:, 0].astype(np.int64); tag = tr[:, 1]
        kind = (tag >> 60).astype(int); sm = ((tag >> 48) & 255).astype(int); item = (tag & 0xffffffff).astype(np.int64)
        t = t - t[kind == 0].min()
        m5 = (kind == 5) & (item < 2**31)
        tab = item >> 22
        key = ((tag >> 32) & 0xffff).astype(np.int64) * 16 + ((tag >> 56) & 15).astype(np.int64)
        dur = {}
        for k in np.unique(key[kind == 4]):
            mk = key == k
            ev = sorted(zip(t[mk], kind[mk], item[mk]))
            st = None
            for tt, kk, ii in ev:
                if kk == 3: st = tt
                elif kk == 4 and st is not None and ii < 2**31: dur.setdefault(int(ii) >> 22, []).append(tt - st); st = None
        print(f"== {names[p]} per table: SMs, items, first end, last end (us), median tap loop (us)")
        for tt in np.unique(tab[m5]):
            mm = m5 & (tab == tt)
            print(f"   table {tt}: SMs {len(np.unique(sm[mm]))}, items {mm.sum()}, ends {t[mm].min()/1e3:.1f} .. {t[mm].max()/1e3:.1f}, taps {np.median(dur.get(int(tt), [0]))/1e3:.2f}")

if os.environ.get("TRACE_FIRST"):
    if os.environ.get("TRACE_FIRST") == "2":  # the same forward twice: is the code still cached?
        B.forward(plan, x, w)
    torch.cuda._sleep(10_000_000)
    B.forward(plan, x, w)
    tr = plan.debug_trace()
    t = tr[:, 0].astype(np.int64); tag = tr[:, 1]
    kind = (tag >> 60).astype(int); item = (tag & 0xffffffff).astype(np.int64)
    key = ((tag >> 32) & 0xffff).astype(np.int64) * 16 + ((tag >> 56) & 15).astype(np.int64)
    t = t - t[kind == 0].min()
    from collections import defaultdict
    first = defaultdict(list)
    for k in np.unique(key[kind == 4]):
        mk = key == k
        ev = sorted(zip(t[mk], kind[mk], item[mk]))
        seq = [(tt, kk, ii) for tt, kk, ii in ev if kk in (2, 3, 4, 5)]
        # first item of this warp: wait start (2), ready (3), taps done (4), end (5)
        d = {kk: tt for tt, kk, ii in seq[:4]}
        it0 = [ii for tt, kk, ii in seq if kk == 3][0]
        if it0 < 2**31 and all(q in d for q in (2, 3, 4, 5)):
            first[int(it0) >> 22].append((d[3], d[4] - d[3], d[5] - d[4]))
        second = [tt for tt, kk, ii in seq if kk == 4]
    print("== forward first item per table: ready at / tap loop / epilogue (us, medians)")
    for tt in sorted(first):
        a = np.array(first[tt])
        print(f"   table {tt}: ready {np.median(a[:,0])/1e3:.2f}  taps {np.median(a[:,1])/1e3:.2f}  epi {np.median(a[:,2])/1e3:.2f}")
    # producers: first load issue and per-table
    m1 = kind == 1
    print("   producer first issue (us):", round(t[m1].min()/1e3, 2), "median first per CTA:",
          round(np.median([t[m1 & (((tag >> 32) & 0xffff) == b)].min() for b in np.unique((tag[m1] >> 32) & 0xffff)])/1e3, 2))

if os.environ.get("TRACE_LAT"):
    for p in (0, 2):
        torch.cuda._sleep(10_000_000)
        if p == 0: B.forward(plan, x, w)
        else: B.backward_weight(plan, x, dy, ws=ws)
        tr = plan.debug_trace()
        t = tr[:, 0].astype(np.int64); tag = tr[:, 1]
        kind = (tag >> 60).astype(int); item = (tag & 0xffffffff).astype(np.int64)
        t = t - t[kind == 0].min()
        iss = {int(i): tt for tt, k, i in zip(t, kind, item) if k == 1}
        rdy = {}
        for tt, k, i in zip(t, kind, item):
            if k == 3 and i < 2**31: rdy.setdefault(int(i), tt)
        lat = np.array([rdy[i] - iss[i] for i in rdy if i in iss])
        iss_t = np.array(sorted(iss.values()))
        print(f"== {names[p]}: load latency (issue -> consumer sees data) median {np.median(lat)/1e3:.2f} us, p10 {np.percentile(lat,10)/1e3:.2f}, p90 {np.percentile(lat,90)/1e3:.2f}; "
              f"issues over time: first {iss_t[0]/1e3:.1f} us, 50% {iss_t[len(iss_t)//2]/1e3:.1f}, last {iss_t[-1]/1e3:.1f}")

if os.environ.get("TRACE_REACT"):
    for p in (0, 2):
        torch.cuda._sleep(10_000_000)
        if p == 0: B.forward(plan, x, w)
        else: B.backward_weight(plan, x, dy, ws=ws)
        tr = plan.debug_trace()
        t = tr[:, 0].astype(np.int64); tag = tr[:, 1]
        kind = (tag >> 60).astype(int); item = (tag & 0xffffffff).astype(np.int64)
        key = ((tag >> 32) & 0xffff).astype(np.int64) * 16 + ((tag >> 56) & 15).astype(np.int64)
        t = t - t[kind == 0].min()
        iss = {int(i): tt for tt, k, i in zip(t, kind, item) if k == 1}
        gaps, waits_after = [], []
        for k in np.unique(key[kind == 4]):
            mk = (key == k)
            seq3 = [(tt, int(i)) for tt, kk, i in sorted(zip(t[mk], kind[mk], item[mk])) if kk == 3 and i < 2**31]
            seq4 = [(tt, int(i)) for tt, kk, i in sorted(zip(t[mk], kind[mk], item[mk])) if kk == 4 and i < 2**31]
            for a in range(len(seq4) - 2):
                rel, nxt = seq4[a][0], seq3[a + 2][1] if a + 2 < len(seq3) else None
                if nxt is not None and nxt in iss: gaps.append(iss[nxt] - rel)
        g = np.array(gaps)
        print(f"== {names[p]}: slot release -> next load issue: median {np.median(g)/1e3:.2f} us, p10 {np.percentile(g,10)/1e3:.2f}, p90 {np.percentile(g,90)/1e3:.2f}")

if os.environ.get("TRACE_PROD"):
    for p in (0, 2):
        torch.cuda._sleep(10_000_000)
        if p == 0: B.forward(plan, x, w)
        else: B.backward_weight(plan, x, dy, ws=ws)
        tr = plan.debug_trace()
        t = tr[:, 0].astype(np.int64); tag = tr[:, 1]
        kind = (tag >> 60).astype(int); item = (tag & 0xffffffff).astype(np.int64)
        blk = ((tag >> 32) & 0xffff).astype(np.int64); wp = ((tag >> 56) & 15).astype(np.int64)
        t = t - t[kind == 0].min()
        d_iss = []
        idle_frac = []
        for b in np.unique(blk[kind == 6])[:40]:
            for pw_ in (0, 1):
                m = (blk == b) & (wp == pw_)
                ev = sorted(zip(t[m], kind[m]))
                last6 = None
                for tt, kk in ev:
                    if kk == 6: last6 = tt
                    elif kk == 1 and last6 is not None: d_iss.append(tt - last6); last6 = None
        d = np.array(d_iss)
        print(f"== {names[p]}: producer detect -> issue median {np.median(d)/1e3:.2f} us, p90 {np.percentile(d,90)/1e3:.2f}, max {d.max()/1e3:.2f}")
        # consumer release (kind 4) -> producer detect (kind 6) for the same pair/slot is harder to pair; report
        # per CTA: number of detects and spacing
        for b in np.unique(blk[kind == 6])[:2]:
            m = (blk == b) & (kind == 6)
            ts = np.sort(t[m]); print("   CTA", b, "detects", len(ts), "spacing median", round(np.median(np.diff(ts))/1e3, 2), "us")
