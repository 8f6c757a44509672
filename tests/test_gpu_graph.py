"""The C-ABI calls are stream-ordered and allocation-free (caller workspace), so a whole CIL
step can be captured into a CUDA graph and replayed: replays on new inputs (copied into the
captured buffers) must equal eager calls bit for bit."""
import numpy as np
import pytest
import torch

import cilgen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cil():
    import paper_2203_14742_b200 as m
    return m


def _radii(A, B, grid, M):
    from oracle import oracle as O
    D = O.distance_matrix(A[:40].numpy(), B[:40].numpy(), grid, 0x1)[0]
    d = D[D > 0]
    return np.quantile(d, np.linspace(0.98, 0.02, M))[None]


@pytest.mark.parametrize("engine_name", ["ENGINE_AUTO", "ENGINE_SIMT"])
def test_features_graph_replay(cil, engine_name):
    dev = torch.device("cuda")
    grid = (2, 32, 32, 0.0)
    P, N, Nt, M = 3, 300, 260, 9
    engine = getattr(cil, engine_name)
    sets = [(cilgen.make_set(81, 2 * i, N, grid[:3]), cilgen.make_set(81, 2 * i + 1, Nt, grid[:3])) for i in range(2 * P)]
    radii = torch.tensor(_radii(sets[0][0], sets[0][1], grid, M), device=dev)
    A = torch.stack([s[0] for s in sets[:P]]).to(dev)
    B = torch.stack([s[1] for s in sets[:P]]).to(dev)
    ws = cil.Workspace()
    counts = torch.empty((P, 1, M), dtype=torch.int64, device=dev)
    y = torch.empty((P, 1, M), dtype=torch.float64, device=dev)
    st = torch.empty((P,), dtype=torch.int32, device=dev)
    kw = dict(engine=engine, ws=ws, counts=counts, y=y, status=st)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cil.features(A, B, grid, cil.L2, radii, **kw)           # warm-up: workspace, attributes
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cil.features(A, B, grid, cil.L2, radii, **kw)
    for rnd in range(2):
        src = sets[rnd * P:(rnd + 1) * P]
        A.copy_(torch.stack([x[0] for x in src]).to(dev))
        B.copy_(torch.stack([x[1] for x in src]).to(dev))
        g.replay()
        torch.cuda.synchronize()
        c_graph, y_graph, s_graph = counts.clone(), y.clone(), st.clone()
        c_eager, y_eager, s_eager = cil.features(A, B, grid, cil.L2, radii, engine=engine)
        torch.cuda.synchronize()
        assert torch.equal(c_graph, c_eager) and torch.equal(y_graph, y_eager) and torch.equal(s_graph, s_eager)
        assert int(c_graph.sum()) > 0


def test_synth_boot_graph_replay(cil):
    """Alg. A2 (bin matrix, tensor-core resample, y~, tail) captured once, replayed."""
    dev = torch.device("cuda")
    grid = (2, 16, 16, 0.0)
    P, N_syn, N_set, n_rep, M = 2, 300, 40, 120, 8
    pools = torch.stack([cilgen.make_set(82, p, N_syn, grid[:3]) for p in range(P)]).to(dev)
    data = cilgen.make_set(82, 50, N_set, grid[:3]).to(dev)
    radii = torch.tensor(np.stack([_radii(pools[p, :150].cpu(), pools[p, 150:].cpu(), grid, M) for p in range(P)]),
                         device=dev)
    draws = [cilgen.boot_draws_a2(83, p, n_rep, N_syn, N_set) for p in range(P)]
    I1 = torch.tensor(np.stack([d[0] for d in draws]), device=dev)
    I2 = torch.tensor(np.stack([d[1] for d in draws]), device=dev)
    J = torch.tensor(np.stack([d[2] for d in draws]), device=dev)
    ws = cil.Workspace()
    out = torch.empty((P, 3), dtype=torch.float64, device=dev)
    st = torch.empty((P,), dtype=torch.int32, device=dev)

    def call():
        cil.synth_loglik_boot(pools, data, N_set, I1, I2, J, grid, cil.L2, radii, ridge=1e-6, ws=ws, out=out,
                              status=st)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    eager = out.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, eager) and int(st.max()) == 0
    # new draws through the same buffers
    draws = [cilgen.boot_draws_a2(84, p, n_rep, N_syn, N_set) for p in range(P)]
    I1.copy_(torch.tensor(np.stack([d[0] for d in draws]), device=dev))
    I2.copy_(torch.tensor(np.stack([d[1] for d in draws]), device=dev))
    g.replay()
    torch.cuda.synchronize()
    replayed = out.clone()
    call()
    torch.cuda.synchronize()
    assert torch.equal(replayed, out) and not torch.equal(replayed, eager)


def test_features_graph_replay_concurrent_engines(cil):
    """All six measures under AUTO: the max family's engine runs on the library's side stream,
    forked from and joined into the captured stream by events — the capture must contain it, and
    replays must equal eager calls bit for bit."""
    from oracle import oracle as O
    dev = torch.device("cuda")
    grid = (2, 24, 24, 0.0)
    P, N, Nt, M = 2, 200, 180, 8
    sets = [(cilgen.make_set(91, 2 * i, N, grid[:3]), cilgen.make_set(91, 2 * i + 1, Nt, grid[:3])) for i in range(2 * P)]
    D = O.distance_matrix(sets[0][0][:40].numpy(), sets[0][1][:40].numpy(), grid, 0x3F)
    radii = torch.tensor(np.stack([np.quantile(d[d > 0], np.linspace(0.97, 0.03, M)) for d in D]), device=dev)
    A = torch.stack([s[0] for s in sets[:P]]).to(dev)
    B = torch.stack([s[1] for s in sets[:P]]).to(dev)
    ws = cil.Workspace()
    counts = torch.empty((P, 6, M), dtype=torch.int64, device=dev)
    y = torch.empty((P, 6, M), dtype=torch.float64, device=dev)
    st = torch.empty((P,), dtype=torch.int32, device=dev)
    kw = dict(engine=cil.ENGINE_AUTO, ws=ws, counts=counts, y=y, status=st)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cil.features(A, B, grid, cil.ALL, radii, **kw)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cil.features(A, B, grid, cil.ALL, radii, **kw)
    for rnd in range(2):
        src = sets[rnd * P:(rnd + 1) * P]
        A.copy_(torch.stack([x[0] for x in src]).to(dev))
        B.copy_(torch.stack([x[1] for x in src]).to(dev))
        counts.zero_()
        g.replay()
        torch.cuda.synchronize()
        c_graph, s_graph = counts.clone(), st.clone()
        c_eager, _, s_eager = cil.features(A, B, grid, cil.ALL, radii, engine=cil.ENGINE_AUTO)
        torch.cuda.synchronize()
        assert torch.equal(c_graph, c_eager) and torch.equal(s_graph, s_eager)
        assert int(c_graph[:, 1].sum()) > 0 and int(c_graph[:, 0].sum()) > 0     # both families counted


def test_first_concurrent_call_inside_capture(cil):
    """On a fresh host thread whose only eager call had no max family, the first call with both
    families (the first to fork onto the side stream, and the first use of the max family's kernels)
    is made inside a graph capture: it must capture and replay correctly."""
    import threading
    from oracle import oracle as O
    res = {}

    def work():
        try:
            dev = torch.device("cuda")
            grid = (2, 16, 16, 0.0)
            A = cilgen.make_set(93, 0, 90, grid[:3]).to(dev)
            B = cilgen.make_set(93, 1, 70, grid[:3]).to(dev)
            D = O.distance_matrix(A[:30].cpu().numpy(), B[:30].cpu().numpy(), grid, 0x3F)
            radii = torch.tensor(np.stack([np.quantile(d[d > 0], np.linspace(0.95, 0.05, 6)) for d in D]), device=dev)
            ws = cil.Workspace()
            counts = torch.empty((1, 6, 6), dtype=torch.int64, device=dev)
            st = torch.empty((1,), dtype=torch.int32, device=dev)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                cil.features(A, B, grid, cil.L2, radii[:1], ws=ws)              # eager, L2 only
            torch.cuda.synchronize()
            ws.get(cil.features_workspace_size(1, 90, 70, grid, cil.ALL, 6, cil.ENGINE_AUTO), dev)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                cil.features(A, B, grid, cil.ALL, radii, ws=ws, counts=counts, status=st)
            counts.zero_()
            g.replay()
            torch.cuda.synchronize()
            c_eager, _, _ = cil.features(A, B, grid, cil.ALL, radii)
            torch.cuda.synchronize()
            res["ok"] = torch.equal(counts, c_eager) and int(st[0]) == 0
        except Exception as e:                       # surfaced by the assertion below
            res["err"] = repr(e)

    t = threading.Thread(target=work)
    t.start()
    t.join()
    assert res.get("ok"), res
