import sys, numpy as np, torch
sys.path.insert(0, '.')
import cilgen, paper_2203_14742_b200 as cil
from oracle import oracle as O
dev = torch.device('cuda')
grid = (2, 16, 16, 0.0)
for (N_syn, N_set, n_rep, M, mask) in [(300, 40, 150, 13, 3), (300, 40, 150, 13, 1), (300, 40, 150, 8, 1), (120, 10, 60, 13, 1), (256, 40, 150, 13, 1), (300, 40, 60, 13, 1)]:
    P = 2
    pools = torch.stack([cilgen.make_set(71, 10 + p, N_syn, grid[:3], n_w=4.6 + 0.3 * p) for p in range(P)])
    data = cilgen.make_set(71, 99, N_set, grid[:3])
    radii, draws = [], []
    for p in range(P):
        D = O.distance_matrix(pools[p, :40].numpy(), pools[p, 40:80].numpy(), grid, mask)
        r = []
        for d in D:
            d = d[d > 0].ravel(); r.append(np.quantile(d, np.linspace(0.98, 0.02, M)))
        radii.append(r)
        draws.append(cilgen.boot_draws_a2(72, p, n_rep, N_syn, N_set))
    radii = torch.tensor(np.array(radii), device=dev)
    I1 = torch.tensor(np.stack([d[0] for d in draws]), device=dev)
    I2 = torch.tensor(np.stack([d[1] for d in draws]), device=dev)
    J = torch.tensor(np.stack([d[2] for d in draws]), device=dev)
    pd = pools.to(dev)
    _, st, Y = cil.synth_loglik_boot(pd, data.to(dev), N_set, I1, I2, J, grid, mask, radii, ridge=1e-5, return_Y=True)
    bins, bst = cil.bin_matrix(pd, pd, grid, mask, radii)
    _, y, rst = cil.resample_counts(bins, I1, I2, M, want_counts=False)
    torch.cuda.synchronize()
    npairs = N_set * (N_syn - N_set)
    a = torch.round(Y[:, :n_rep] * npairs).long().cpu().numpy(); b = torch.round(y * npairs).long().cpu().numpy()
    d = a - b
    nz = np.argwhere(d != 0)
    print((N_syn, N_set, n_rep, M, mask), 'ndiff', len(nz), 'of', d.size, 'sym', bool(torch.equal(bins, bins.transpose(2, 3))))
    if len(nz):
        print('  p set', sorted(set(nz[:, 0])), 'k set', sorted(set(nz[:, 1]))[:20], 'col set', sorted(set(nz[:, 2])))
        print('  sample diffs', [(tuple(i), int(d[tuple(i)]), int(b[tuple(i)])) for i in nz[:8]])
