"""Test infrastructure (may use oracle/; not collected by pytest): one-off full-scale check, every BASELINE source of the
given configs, top-down and direction-optimising, levels bit-exact and parents by certificate."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, graphgen, oracle, paper_2209_08764_b200 as pkg
for cfg in sys.argv[1:]:
    g = graphgen.make_config(cfg)
    ro = torch.from_numpy(g.row_offsets).cuda(); col = torch.from_numpy(g.col_indices).cuda()
    hs = {"td": pkg.S3BFS(ro, col), "do": pkg.S3BFS(ro, col, pkg.Options(direction=1))}
    bad = 0
    t0 = time.time()
    for s in g.sources:
        ref, _ = oracle.bfs(g.row_offsets, g.col_indices, int(s))
        for k, h in hs.items():
            lv, pa = h.run(int(s)); torch.cuda.synchronize()
            lvn, pan = lv.cpu().numpy(), pa.cpu().numpy()
            ok = np.array_equal(lvn, ref)
            code, _ = oracle.check_bfs(g.row_offsets, g.col_indices, int(s), lvn, pan)
            if not ok or code != 0:
                bad += 1; print("MISMATCH", cfg, k, s, ok, code, flush=True)
    print(f"{cfg}: {len(g.sources)} sources x (td, do): mismatches {bad} ({time.time()-t0:.0f} s)", flush=True)
