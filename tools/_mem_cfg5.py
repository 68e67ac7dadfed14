import sys; sys.path.insert(0, '.')
import torch, bench, paper_2006_06052_b200 as amg
ptr, col, val, b = bench.make_problem(5, 256, 0, 256 ** 3)
S = amg.Solver(amg.BSR.from_numpy(ptr, col, val), bench.params_for(amg, 5))
del val
print(S.memory_report())
bd = torch.as_tensor(b, device="cuda"); x = torch.zeros_like(bd)
rep = S.solve(bd, x, 1e-8); print(rep.iters, rep.relres_true, rep.converged)
