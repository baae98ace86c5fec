import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2605_05696_b200 import chunking
rng=np.random.default_rng(0)
streams=[rng.integers(0,2**32,size=32900,dtype=np.uint64).astype(np.uint32) for _ in range(8)]
t=chunking.cdc_chunk_batch(streams, chunking.ChunkerParams(), [set()]*8); torch.cuda.synchronize()
t=chunking.cdc_chunk_batch(streams, chunking.ChunkerParams(), [set()]*8); torch.cuda.synchronize()
