"""Encode the C1 fixture (sphere 128^3, ACCEPT_CONFIG, fp16 container) with the reference.

Run once in the build container (~7 min on 8 cores); writes /tmp/gw/c1.nvdb for make_golden.py --c1."""
import time, pickle, numpy as np
from svcodec.config import TrainConfig
from svcodec.container import serialize_container, deserialize_container
from svcodec.encoder import encode
from svcodec.decoder import decode_full
from svcodec.procgen import SphereSpec, gen_sphere_sdf
g = gen_sphere_sdf(SphereSpec(center=(63.5,63.5,63.5), radius=61.0, voxel_size=1.0, half_width=3.0))
cfg = TrainConfig(subdomain_size=512, l1_net=(3, 48), tile_net=None, l0_net=(3, 96),
    voxel_net=(3, 96), activation="sine", frequency=3.0, ffm_scale=5.0,
    ffm_size=192, lr=1e-3, decay=0.975, interval=100.0, max_epochs=800,
    sample_interval=1, batch_size=65536, significance_threshold=0.0,
    strict_topology=False, seed=4242)
t=time.time(); c = encode(g, cfg, weight_precision=16); print("encode", time.time()-t, flush=True)
blob = serialize_container(c)
open('/tmp/gw/c1.nvdb','wb').write(blob)
c2 = deserialize_container(blob)
t=time.time(); d = decode_full(c2); print("decode", time.time()-t, flush=True)
pickle.dump({'grid': g, 'decoded': d}, open('/tmp/gw/c1_grids.pkl','wb'))
print("done")
