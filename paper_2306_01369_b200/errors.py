"""Exception types of the reference API (scene.py:35-45, contact.py:29-30)."""


class SceneError(ValueError):
    pass


class SceneParseError(SceneError):
    pass


class ValidationError(SceneError):
    pass


class SolverError(RuntimeError):
    pass
