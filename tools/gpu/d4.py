import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_2210_06160_b200 as rt
from paper_2210_06160_b200 import geometry as G
for name in ["sphere_plane","sphere","box_spheres","big_sphere"]:
    sc=rt.get_scene(name); b=sc.view(0).bvh
    n4=b.search_nodes4
    raw=b.search.cpu().numpy().view(np.uint8)
    nodes4=raw[-n4*128:].reshape(n4,128) if n4 else None
    print(name, "n4", n4, "depth4", G._depth4(nodes4) if n4 else None)
