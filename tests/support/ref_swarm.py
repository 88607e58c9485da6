"""TEST-ONLY: stand up the reference's OWN simulated swarm
(`swarmpipe.swarm.build_sim_swarm`: DirectoryBoard + BlockServer + SimNetwork +
SwarmClient, SP/swarm.py:52-94) with the B200 engine as the server payload
engine and the GPU client head as the client payload engine.

This is the drop-in recipe of SURVEY.md §7 step 2: the reference's
`RealServerEngine` / `RealClientEngine` names are rebound for the duration of
the build, nothing else of the reference is touched.  `init_model` is rebound
too when the model is not the reference's own (Llama / BLOOM shapes): the B200
engine and head regenerate their weights on the GPU from the seed, so the
reference's numpy copy is never needed.
"""

from __future__ import annotations

import contextlib

_HEADS: dict = {}


def gpu_client_engine_class(swarmpipe):
    """A `RealClientEngine` subclass (SwarmClient.beam_generate requires one,
    SP/client.py:599) whose payload is `paper_2312_08361_b200.head.ClientHead`."""
    from paper_2312_08361_b200.head import ClientHead

    class GpuClientEngine(swarmpipe.client.RealClientEngine):
        def __init__(self, config, client_params=None, device: int = 0):
            self.config = config
            key = (repr(config), device)
            if key not in _HEADS:
                _HEADS[key] = ClientHead(config, device)
            self.head = _HEADS[key]

        def embed_array(self, tokens):
            return self.head.embed_array(tokens)

        def pick(self, final_rows, mode, rng, top_k):
            return self.head.pick(final_rows, mode, rng, top_k)

        def logits(self, rows):
            return self.head.logits(rows)

    return GpuClientEngine


@contextlib.contextmanager
def rebound(swarmpipe, engine_factory, client_engine=True, skip_numpy_init=False):
    """Rebind the reference's engine names (SP/swarm.py:16, SP/server.py,
    SP/__init__.py:60) while the swarm is built."""
    import swarmpipe.server as srv
    import swarmpipe.swarm as sw
    saved = (sw.RealServerEngine, srv.RealServerEngine, swarmpipe.RealServerEngine,
             sw.RealClientEngine, sw.init_model)
    sw.RealServerEngine = srv.RealServerEngine = swarmpipe.RealServerEngine = engine_factory
    if client_engine:
        sw.RealClientEngine = gpu_client_engine_class(swarmpipe)
    if skip_numpy_init:
        sw.init_model = lambda model: (None, None)
    try:
        yield
    finally:
        (sw.RealServerEngine, srv.RealServerEngine, swarmpipe.RealServerEngine,
         sw.RealClientEngine, sw.init_model) = saved


def build_gpu_swarm(swarmpipe, model, *, engine_for=None, **kw):
    """`build_sim_swarm(model, **kw)` with B200 server engines.

    engine_for(stage, replica) -> engine places each server's engine (several
    GPUs); default: one B200ServerEngine per server over the process-wide
    shared span of this model (SP/swarm.py:72-74 shares the blocks likewise).
    The client factory of the returned SimSwarm uses the GPU head."""
    from paper_2312_08361_b200.config import SpanConfig
    from paper_2312_08361_b200.engine import B200ServerEngine
    replicas = kw.get("replicas", 2)
    made = []

    def factory(config, blocks=None):
        i = len(made)
        stage, replica = divmod(i, replicas)   # build order: stage-major (SP/swarm.py:80-82)
        eng = engine_for(stage, replica) if engine_for else B200ServerEngine(config, blocks)
        made.append(eng)
        return eng

    with rebound(swarmpipe, factory, skip_numpy_init=isinstance(model, SpanConfig)):
        swarm = swarmpipe.swarm.build_sim_swarm(model, **kw)
    # SimSwarm.client() resolves RealClientEngine at call time: bind the GPU head
    # for this swarm's clients
    GpuClient = gpu_client_engine_class(swarmpipe)
    orig_client = swarm.client

    def client(name=None, **ckw):
        import swarmpipe.swarm as sw
        saved = sw.RealClientEngine
        sw.RealClientEngine = GpuClient
        try:
            return orig_client(name, **ckw)
        finally:
            sw.RealClientEngine = saved

    swarm.client = client
    return swarm
