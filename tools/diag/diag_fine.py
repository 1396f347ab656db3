import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import paper_2503_03479_b200 as xa
from oracle.oracle import Oracle
port=Oracle("port")
for p,size in (([0.3,1.414,-0.9,0.8,0,0],256),([0.0,1.414,0.5,1.0,0,0],320)):
    img = port.make_texture(size, size - 32, 12 if size == 256 else 4)
    tgt = port.warp(img, port.affine_from_params(p), "lanczos")[0]
    params = xa.AffineParams(psi=0.0, tilt=p[1], phi=p[2], scale=p[3])
    got, fwd = xa.fine_correspondences(img, tgt, params, max_points=800)
    pr=[0.0,p[1],p[2],p[3],0,0]
    filt = port.antialias_tilt(img, p[1], p[2])
    gf = xa.antialias_tilt(img, p[1], p[2])
    print("filt diff", np.abs(gf-filt).max())
    wimg, _, _, pfwd = port.warp(filt, port.simulation_from_params(pr), "lanczos", 4)
    gw = xa.warp_lanczos(filt, xa.simulation_from_params(params), 4)
    print("view diff", np.abs(gw.image-wimg).max(), np.mean(gw.image!=wimg))
    back = port.invert(pfwd)
    kd = port.detect_dog(wimg, 800); gk = xa.detect_dog_keypoints(gw.image, 800)
    print("kps", len(kd), len(gk))
    kps = port.filter_to_content(kd, back, img.shape[1], img.shape[0], 4.0)
    wk, wd = port.describe_gradient(wimg, kps)
    tk, td = port.describe_gradient(tgt, port.detect_dog(tgt, 800))
    gtk, gtd = xa.fine_features(tgt, 800)
    print("tgt kps", len(tk), len(gtk), np.array_equal(np.sort(tk[:,:2],0), np.sort(gtk[:,:2],0)))
    m = port.match_ratio(wd, td, 0.75)
    want=[]
    for r in m:
        x, y = xa.map_point(back, float(wk[r["idx_a"], 0]), float(wk[r["idx_a"], 1]))
        want.append((x, y, float(tk[r["idx_b"], 0]), float(tk[r["idx_b"], 1])))
    want=np.array(want)
    print(len(want), len(got))
    for w in want:
        d=np.abs(got[:,:4]-w).max(1)
        print(w, d.min())
