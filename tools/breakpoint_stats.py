import sys, numpy as np, time
sys.path.insert(0, '/root/repo')
from oracle import splitplan_oracle as O
NEG = -np.inf

def shift(row, h, W):
    c, v = row
    c = c + h
    m = c <= W
    return c[m], v[m]

def vmax(a, b):
    # pointwise max of two monotone step functions given as (cols asc, vals asc)
    ca, va = a; cb, vb = b
    cols = np.union1d(ca, cb)
    ia = np.searchsorted(ca, cols, side='right') - 1
    ib = np.searchsorted(cb, cols, side='right') - 1
    va2 = np.concatenate([[NEG], va]); vb2 = np.concatenate([[NEG], vb])
    xa = va2[ia + 1]
    xb = vb2[ib + 1]
    x = np.maximum(xa, xb)
    keep = np.ones(len(x), bool)
    keep[1:] = x[1:] != x[:-1]
    keep &= x != NEG
    return cols[keep], x[keep]

def sparse_tables(inst):
    L = len(inst["r"]); W = O.effective_budget(inst)
    z = (np.array([0], np.int64), np.array([0.0]))
    e = (np.zeros(0, np.int64), np.zeros(0))
    C, S = (z, e) if inst["sac"] else (e, z)
    rows = [(C, S)]
    for k in range(L):
        i, s, u, d = (int(inst[x][k]) for x in "isud")
        cm = vmax(shift(C, i, W), shift(S, i + d, W))
        cv = cm[1] + inst["r"][k]
        keep = np.ones(len(cv), bool); keep[1:] = cv[1:] != cv[:-1]
        Cn = (cm[0][keep], cv[keep])
        Sn = vmax(shift(S, s, W), shift(C, s + u, W))
        C, S = Cn, Sn
        rows.append((C, S))
    return rows, W

def densify(row, W):
    c, v = row
    out = np.full(W + 1, NEG)
    for t in range(len(c)):
        out[c[t]:(c[t+1] if t + 1 < len(c) else W + 1)] = v[t]
    return out

if __name__ == "__main__" and len(sys.argv) == 1:
    from paper_2410_10759_b200 import workloads as Wk
    layers = O.preset_layers("gpt2-24")
    req, _ = Wk.cfg2(40, 2000)
    mx = []
    for k in range(40):
        s = int(req["seq_len"][k])
        r, cs, ss, tau = O.profile_arrays(layers, s, req["client_fps"][k], req["server_fps"][k])
        inst = O.instance_from_profile(r, cs, ss, tau, req["uplink_bps"][k], req["downlink_bps"][k], 0.01, req["deadline_s"][k], req["unit_s"][k])
        rows, W = sparse_tables(inst)
        mx.append(max(max(len(a[0]), len(b[0])) for a, b in rows))
        if k < 6:
            C, S = O.dp_tables(inst)
            for kk in range(len(rows)):
                assert np.array_equal(densify(rows[kk][0], W), C[kk]), (k, kk)
                assert np.array_equal(densify(rows[kk][1], W), S[kk]), (k, kk)
    print("cfg2 max breakpoints per row:", sorted(mx))

def stats(name, insts, check=0):
    mx = []
    for n, inst in enumerate(insts):
        rows, W = sparse_tables(inst)
        mx.append(max(max(len(a[0]), len(b[0])) for a, b in rows))
        if n < check:
            C, S = O.dp_tables(inst)
            for kk in range(len(rows)):
                assert np.array_equal(densify(rows[kk][0], W), C[kk]) and np.array_equal(densify(rows[kk][1], W), S[kk])
    mx = np.array(mx)
    print(name, "n", len(mx), "median", np.median(mx), "p99", np.percentile(mx, 99), "max", mx.max())

def run_more():
    from paper_2410_10759_b200 import workloads as Wk
    req, _ = Wk.cfg3(60, 3)
    layers = [dict(kind="embedding", hidden_dim=4096, out_dim=32000, seq_divisor=1)]
    from paper_2410_10759_b200 import cost_model as cm
    insts = []
    L3 = Wk.llama2_7b_layers()
    import dataclasses
    for k in range(60):
        s = int(req["seq_len"][k])
        prof = cm.profile(cm.ModelSpec("llama", L3) if hasattr(cm, "ModelSpec") else None, cm.DeviceSpec("c", req["client_fps"][k]), cm.DeviceSpec("s", req["server_fps"][k])) if False else None
    return

if __name__ == "__main__" and len(sys.argv) > 1:
    import json
    z = np.load('/root/repo/tests/golden/battery_float.npz')
    off = z["off"]
    insts = [dict(i=z["i"][off[k]:off[k+1]], s=z["s"][off[k]:off[k+1]], u=z["u"][off[k]:off[k+1]], d=z["d"][off[k]:off[k+1]], r=z["r"][off[k]:off[k+1]], budget=int(z["budget"][k]), sac=bool(z["sac"][k])) for k in range(min(200, len(off)-1))]
    stats("battery_float", insts, check=50)
    rng = np.random.default_rng(5)
    L = 2000; Wc = 200000
    inst = dict(i=rng.integers(0, 201, L), s=rng.integers(0, 201, L), u=rng.integers(0, 201, L), d=rng.integers(0, 201, L), r=rng.integers(0, 101, L).astype(float), budget=Wc, sac=True)
    t=time.time(); rows, W = sparse_tables(inst); 
    print("cfg5-like L=2000 W=2e5 breakpoints per row: max", max(max(len(a[0]), len(b[0])) for a, b in rows), "last", len(rows[-1][0][0]), time.time()-t)
