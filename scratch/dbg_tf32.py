import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from test_gpu_gemm import run, matmul_doc
for (m,k,n,tb) in [(128,32,128,False),(128,32,128,True),(128,64,128,False),(256,512,384,False),(1024,4096,1024,False),(128,128,256,False)]:
    a,b,c,names = run(matmul_doc(m,k,n,tb,dtype="f32"))
    A=a.astype(np.float64); B=b.astype(np.float64)
    ref = A @ (B.T if tb else B)
    err = np.abs(c-ref).max()/np.abs(ref).max()
    # compare with 1xTF32-ish estimate
    bad = np.argwhere(np.abs(c-ref) > 1e-4*np.abs(ref).max())
    print(m,k,n,tb, names, f"err={err:.3e}", "nbad", len(bad), bad[:3].tolist(), c.ravel()[:3], ref.ravel()[:3])
