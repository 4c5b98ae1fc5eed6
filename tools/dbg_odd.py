import sys
import torch
sys.path.insert(0, ".")
import paper_2011_02436_b200 as rb

def inputs(L, m, n=4000, d=16):
    x, t = rb.synth_classification(n, d, m, seed=51, teacher_seed=52)
    p = rb.ElmParams(d, L, m, 53)
    hid = rb.init_hidden(p)
    X, T = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
    W = torch.from_numpy(hid.weights).cuda()
    B = torch.from_numpy(hid.biases.reshape(-1)).cuda()
    return X, T, W, B

for L, m in ((400, 5), (201, 2)):
    X, T, W, B = inputs(L, m)
    M = L + m
    outs = []
    for rep in range(4):
        g = torch.empty((M, M + (rep % 2)), dtype=torch.float64, device="cuda")[:, :M]
        rb.gram_stage_device_aug(X, T, W, B, g)
        outs.append(g.clone())
    print(L, m, "repeat-equal", [torch.equal(outs[0], o) for o in outs[1:]],
          "maxdiff", max((outs[0] - o).abs().max().item() for o in outs[1:]))
    g2 = outs[0].clone()
    rb.gram_stage_device_aug(X, T, W, B, g2, accumulate=True)
    print(L, m, "acc==2g", torch.equal(g2, 2 * outs[0]))
    h = torch.sigmoid(X @ W + B)
    gh = torch.empty((L, L), dtype=torch.float64, device="cuda")
    rb.gram_device(h, gh)
    print(L, m, "gram_device close", torch.allclose(gh, outs[0][:L, :L], rtol=1e-12, atol=1e-9))
