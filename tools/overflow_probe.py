import sys; sys.path.insert(0,'/root/repo')
import numpy as np, torch
from paper_1710_07745_b200 import canny
import oracle.oracle as O
for low, high in [(5.0,100.0),(2.0,400.0)]:
    rng = np.random.default_rng(int(low*10+high))
    frames = rng.integers(0,256,size=(1,2048,2048),dtype=np.uint8)
    w = O.gaussian_weights(0.6, radius=1)
    ws = canny.new_workspace(1,2048,2048)
    lab, fin = canny.canny_u8(torch.from_numpy(frames).cuda(), w, low, high, ws=ws)
    torch.cuda.synchronize()
    h = ws[:64].cpu().numpy()
    u32 = h.view(np.uint32); u64 = h.view(np.uint64)
    print(low, high, 'fix_count', u64[4], 'overflow', u32[12], 'plist_ovf', u32[13], 'dense', u32[14], 'node_ovf', u32[15])

# fix-list overflow (threshold ties) and node-list overflow (large noise)
rng = np.random.default_rng(3)
blk = rng.choice(np.array([0, 16], np.uint8), size=(512, 512))
frames = np.kron(blk, np.ones((4, 4), np.uint8))[None]
for low, high in [(48.0, 48.0), (16.0, 48.0)]:
    ws = canny.new_workspace(1, 2048, 2048)
    canny.canny_u8(torch.from_numpy(frames).cuda(), np.array([0.25, 0.5, 0.25]), low, high, ws=ws)
    torch.cuda.synchronize()
    h = ws[:64].cpu().numpy(); u32 = h.view(np.uint32); u64 = h.view(np.uint64)
    print('ties', low, high, 'fix_count', u64[4], 'overflow', u32[12], 'plist_ovf', u32[13], 'dense', u32[14], 'node_ovf', u32[15])
rng = np.random.default_rng(8192)
frames = rng.integers(0, 256, size=(1, 8192, 8192), dtype=np.uint8)
ws = canny.new_workspace(1, 8192, 8192)
canny.canny_u8(torch.from_numpy(frames).cuda(), O.gaussian_weights(0.6, radius=1), 5.0, 60.0, ws=ws)
torch.cuda.synchronize()
h = ws[:64].cpu().numpy(); u32 = h.view(np.uint32); u64 = h.view(np.uint64)
print('noise8k fix_count', u64[4], 'overflow', u32[12], 'plist_ovf', u32[13], 'dense', u32[14], 'node_ovf', u32[15])
