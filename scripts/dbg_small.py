import sys, ctypes, numpy as np, torch
sys.path.insert(0, '.')
import graphgen, oracle
import paper_2209_08764_b200.s3bfs as S
S.LIB_PATH = sys.argv[1]
S._build.LIB = sys.argv[1]
lib = S.load(build_if_missing=False)
g = graphgen.from_edges(60, [(i, i + 1) for i in range(59)])
ro = torch.from_numpy(g.row_offsets).cuda(); col = torch.from_numpy(g.col_indices).cuda()
h = S.s3bfs_create(ro, col, S.Options(tier0_max_edges=-1, cluster_max_edges=-1, loop_mode=2))
lv = torch.empty(60, dtype=torch.int32, device='cuda'); pa = torch.empty_like(lv)
rc = lib.s3bfs_run(h, 0, lv.data_ptr(), pa.data_ptr(), torch.cuda.current_stream().cuda_stream)
print("rc", rc)
out = (ctypes.c_uint64 * 4)()
print("dbg rc", lib.s3bfs_debug_timeline(h, out), [hex(x) for x in out])
print(lv.cpu().numpy()[:10])
st = S.s3bfs_get_level_stats(h)
print(st[:5])
