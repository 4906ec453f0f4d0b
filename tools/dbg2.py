import numpy as np, torch, sys
sys.path.insert(0,'.')
from oracle import packkv_oracle as O
from paper_2512_24449_b200 import bitpack_codec as C, quantizer as Q
rng=np.random.default_rng(0)
rows,cols,k=16,4,16
q=np.zeros((1,rows,cols),np.int64)
for sc in [rng.uniform(0.01,2,(1,rows)).astype(np.float32), np.arange(1,17,dtype=np.float32)[None]*0.37, np.full((1,rows),1.0009765625,np.float32)]:
    zp=np.zeros((1,rows),np.float32)
    qb=Q.QuantBlock(torch.from_numpy(q.astype(np.int32)).to(torch.uint16).cuda(), torch.from_numpy(sc).cuda(), torch.from_numpy(zp).cuda(), 0)
    b=C.encode_blocks(qb,k,0)[0].to_bytes()
    ref=O.encode_block(O.QuantBlock(q[0],sc[0],zp[0],0),k,0,0)
    print('ours', [hex(x) for x in np.frombuffer(b[18:82],np.uint16)[0::2]])
    print('ref ', [hex(x) for x in np.frombuffer(ref[18:82],np.uint16)[0::2]])
d=C.decode_block(C.PackedBlock.from_bytes(ref)); print('dec scale', d.scale.cpu().numpy()[:4])
