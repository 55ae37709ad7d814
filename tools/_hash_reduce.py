import os, sys, hashlib
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2002_05018_b200 import fem3d, subdomain
model = fem3d.build_model(fem3d.config2())
systems = fem3d.subdomain_systems(model)
red = subdomain.reduce_domains(systems)
h = hashlib.sha256()
for (K, g), s in zip(red, systems):
    h.update(np.ascontiguousarray(np.asarray(K)).tobytes()); h.update(np.ascontiguousarray(np.asarray(g)).tobytes())
    h.update(s._d3m_X.cpu().numpy().tobytes())
print("cfg2 reduce sha256", h.hexdigest())
