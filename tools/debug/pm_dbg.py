import numpy as np, torch, sys, math
sys.path.insert(0, '.')
from paper_2510_03557_b200 import gravity as G
from paper_2510_03557_b200.box import BoxGeometry
g = dict(np.load('tests/golden/pm.npz'))
box = BoxGeometry(1.0); n = int(g['grid_n'])
split = G.ForceSplit(r_s=float(g['r_s']), r_cut=float(g['r_cut']))
rho = torch.from_numpy(g['rho']).cuda()
rk = torch.fft.rfftn(rho)
rk_np = np.fft.rfftn(g['rho'])
print('rfftn diff', np.abs(rk.cpu().numpy() - rk_np).max(), np.abs(rk_np).max(), rk.dtype, rk.is_contiguous(), rk.stride())
fields, pot = G.solve_long_range_device(rho, split, box, True, 'optimal')
print('pot diff', np.abs(pot.cpu().numpy() - g['optimal_pot']).max(), np.abs(g['optimal_pot']).max())
phik_np = -(4*math.pi) * rk_np * g['d_opt']; phik_np[0,0,0] = 0
pot_np = np.fft.irfftn(phik_np, s=(n,n,n))
print('pot via numpy from d_opt', np.abs(pot_np - g['optimal_pot']).max())
k1 = 2*math.pi*np.fft.fftfreq(n, d=1/n); k3 = 2*math.pi*np.fft.rfftfreq(n, d=1/n)
fx_np = np.fft.irfftn(-1j*k1[:,None,None]*phik_np, s=(n,n,n))
print('fx numpy', np.abs(fx_np - g['optimal_fields'][0]).max(), 'ours', np.abs(fields[0].cpu().numpy() - g['optimal_fields'][0]).max())
print(fields[0].shape, fields[0].stride(), fields[0].dtype)
