import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19693_b200 import he_api
from paper_2506_19693_b200 import bootstrap_consts as BC
from paper_2506_19693_b200.backend import GpuCiphertext
from paper_2506_19693_b200.scheme import SchemeParams
from paper_2506_19693_b200.bootstrap import Bootstrapper, bootstrap_rotations
logn = int(sys.argv[1]) if len(sys.argv) > 1 else 12
n = 1 << logn; L = 24; slots = n // 2
params = SchemeParams(poly_degree=n, modulus_chain=(60,) + (45,) * 8 + (60,) * 16 + (660,), scale_bits=45, level=L, bootstrap_depth=16)
cust = he_api.keygen(params, bootstrap_rotations(params), backend="ckks", rng_seed=1, prime_layout="bootstrap", dnum=3, secret_hw=192, conjugation_key=True)
be = cust.backend; ch = be.chain
bs = Bootstrapper(be)
rng = np.random.default_rng(0)
v = rng.uniform(-1, 1, slots)
ct = be._encrypt_values(v, 0)
q0 = ch.entry_products[0]
ph0 = ch.to_f64(be._phase(ct), 1)[0].cpu().numpy()
raised = be.mod_raise(ct)
phr = ch.to_f64(be._phase(raised), be._limbs(L))[0].cpu().numpy()
def dec(x): return be.decrypt_complex(GpuCiphertext(x[0], x[1]), scale=x[2])
x = (raised.data, raised.level, float(q0))
for t, plan in enumerate(bs.cts_plans):
    x = bs._linear(x, plan, ("cts", t))
cp = (phr[:slots] + 1j * phr[slots:]) / (2 * q0 * (bs.K + 1))
bits = slots.bit_length() - 1
idx = np.arange(slots); rev = np.zeros_like(idx)
for b in range(bits): rev |= ((idx >> b) & 1) << (bits - 1 - b)
print("cts level", x[1], "scale 2^%.3f" % np.log2(x[2]), "err", np.max(np.abs(dec(x) - cp[rev])), "mag", np.max(np.abs(cp)))
data, lvl, sc = x; m = be._limbs(lvl)
conj = be.rotate_data(data, lvl, bs.conj)
re = (ch.add(data, conj, m), lvl, sc)
xre = (2*cp[rev]).real
print("re err", np.max(np.abs(dec(re).real - xre)), "imag part max", np.max(np.abs(dec(re).imag)))
T = bs._chebyshev_basis(re)
for k in [1,2,3,4,8,15,16,32,64]:
    tk = np.cos(k*np.arccos(np.clip(xre,-1,1)))
    print("T", k, "level", T[k][1], "scale 2^%.4f" % np.log2(T[k][2]), "err %.3e" % np.max(np.abs(dec(T[k]).real - tk)))
y = bs._eval_cheb(bs.cheb, T, bs._cheb_level(T, len(bs.cheb) - 1), re[2])
f = BC.evalmod_function(bs.K, bs.r)(xre)
print("cheb level", y[1], "err %.3e" % np.max(np.abs(dec(y).real - f)))
for _ in range(bs.r):
    y = bs._add_const(bs._double(bs._mul(y, y)), -1.0)
s = np.sin(2*np.pi*(bs.K+1)*xre)
print("evalmod level", y[1], "err %.3e" % np.max(np.abs(dec(y).real - s)), "target mag %.3e" % np.max(np.abs(s)))
c = ph0
want = 2*np.pi*(c[:slots])/q0
print("sin vs 2pi c/q0: %.3e" % np.max(np.abs(s - want[rev])))
