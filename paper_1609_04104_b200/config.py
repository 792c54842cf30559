"""``ConfigError`` (`pkg/src/tensortrack/config.py:19`), the reference's configuration exception
(SURVEY §8(b) error conventions). The experiment-configuration loader itself is harness code outside
the hot path; engine arguments that are out of range raise this subclass of ValueError."""

__all__ = ["ConfigError"]


class ConfigError(ValueError):
    """Raised for malformed or inconsistent experiment configuration."""
