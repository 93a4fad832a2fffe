import sys, time; sys.path.insert(0, '.')
import bench
from paper_2309_04671_b200 import DeviceTarget, corpus
for builder, shape in (("star3d4r_norm", (512, 512, 512)), ("wave", (512, 512, 512)), ("jacobi7", (512,512,512))):
    bound, decls = corpus.config_target(builder, shape, 4, "f32")
    names = list(decls)
    dt = DeviceTarget({n: bench._decl_grid(d) for n, d in decls.items()}, names, precision="exact")
    bench.fill_device(dt, names, shape, builder)
    dt.set_program(bound.stmts[0].body)
    dt.run(2); dt.sync(); dt.run(4); dt.sync()
    ms = dt.elapsed_ms() / 4
    n = shape[0]*shape[1]*shape[2]
    print(builder, "exact", round(ms, 3), "ms/step", round(n / ms / 1e6, 1), "GPts/s")
    dt.close()
