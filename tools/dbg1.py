import numpy as np, torch, sys
sys.path.insert(0,'.')
from oracle import packkv_oracle as O
from paper_2512_24449_b200 import bitpack_codec as C, quantizer as Q
rng=np.random.default_rng(0)
for (rows,cols,k) in [(16,4,16),(64,128,2),(64,128,16)]:
    q=np.zeros((2,rows,cols),np.int64); q[1]=rng.integers(0,4,(rows,cols))
    sc=rng.uniform(0.01,2,(2,rows)).astype(np.float32); zp=np.zeros((2,rows),np.float32)
    qb=Q.QuantBlock(torch.from_numpy(q.astype(np.int32)).to(torch.uint16).cuda(), torch.from_numpy(sc).cuda(), torch.from_numpy(zp).cuda(), 0)
    blocks=C.encode_blocks(qb,k,0)
    for i in range(2):
        ref=O.encode_block(O.QuantBlock(q[i],sc[i],zp[i],0),k,0,0); got=blocks[i].to_bytes()
        print(rows,cols,k,i,len(ref),len(got), ref==got)
        if ref!=got:
            a=np.frombuffer(ref,np.uint8); b=np.frombuffer(got,np.uint8); n=min(len(a),len(b)); d=np.nonzero(a[:n]!=b[:n])[0]
            print(' first diffs', d[:10], 'hdr', O.header_bytes(rows,cols,k), a[d[:6]], b[d[:6]])
