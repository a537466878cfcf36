import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import datagen, oracle, paper_1803_04120_b200 as sj
d, eps = 2, 0.4
pts = datagen.clustered_small(6000, d, seed=d, sigma=0.3)
want = oracle.brute_force(pts, eps)
idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
print("cells", idx.n_cells, "mode/geom", idx.geometry()["dir_k"])
def chk(tag, r):
    got = r.to_numpy()
    extra = np.setdiff1d(got, want); miss = np.setdiff1d(want, got)
    dup = len(got) - len(np.unique(got))
    print(f"{tag}: got={len(got)} want={len(want)} extra={len(extra)} miss={len(miss)} dup={dup} retries={r.stats['retries']} batches={r.n_batches}")
for dense in (True, False):
    for unicomp in (True, False):
        chk(f"dense={dense} uni={unicomp}", sj.self_join(idx, dense_cells=dense, unicomp=unicomp))
for cap in (5000, 300):
    for host in (False, True):
        for dense in (True, False):
            chk(f"cap={cap} host={host} dense={dense}", sj.self_join(idx, batch_capacity_pairs=cap, result_on_host=host, dense_cells=dense))
