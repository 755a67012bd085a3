"""Exception types of the drop-in API. Same names and meaning as the reference's
(fedforge params.py:39, fedopt.py:22, trainer.py:36-41, model.py:23, data.py:16);
defined here, not imported from the reference."""


class ParamError(ValueError):
    """Invalid parameter-vector construction or arithmetic (incl. non-finite results)."""


class AggregationError(RuntimeError):
    """Protocol violation while accumulating client updates."""


class RoundFailedError(RuntimeError):
    """Local training aborted (non-finite loss or injected crash)."""

    def __init__(self, client_id: int, message: str):
        super().__init__(f"client {client_id}: {message}")
        self.client_id = client_id


class TokenRangeError(ValueError):
    """A batch contains a token id outside the model vocabulary."""


class DataError(ValueError):
    pass


class UnsupportedShapeError(ParamError):
    """The model shape is outside what the sm_100a kernels implement (no CPU fallback)."""
