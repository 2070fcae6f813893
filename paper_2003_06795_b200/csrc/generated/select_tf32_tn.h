#ifndef SELECT_TF32_TN_H
#define SELECT_TF32_TN_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tn_config;

static inline select_tf32_tn_config select_tf32_tn(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(1087)) {
        if (m < INT64_C(70960)) {
            if (n < INT64_C(351)) {
                if (m < INT64_C(8870)) {
                    if (k < INT64_C(444)) {
                        if (k < INT64_C(79)) {
                            if (m < INT64_C(2218)) {
                                if (m < INT64_C(224)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(28)) {
                                    if (m < INT64_C(4435)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (m < INT64_C(4435)) {
                                        if (k < INT64_C(46)) {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(46)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (n < INT64_C(46)) {
                                    if (k < INT64_C(118)) {
                                        if (m < INT64_C(4435)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(2218)) {
                                            if (m < INT64_C(1109)) {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(167)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(2218)) {
                                        if (n < INT64_C(79)) {
                                            if (m < INT64_C(1109)) {
                                                if (k < INT64_C(272)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(79)) {
                                            if (m < INT64_C(4435)) {
                                                if (k < INT64_C(272)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (n < INT64_C(203)) {
                                if (k < INT64_C(744)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(139)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (n < INT64_C(287)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(287)) {
                                if (k < INT64_C(992)) {
                                    if (n < INT64_C(79)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(744)) {
                                            if (k < INT64_C(544)) {
                                                if (m < INT64_C(2218)) {
                                                    if (n < INT64_C(182)) {
                                                        if (m < INT64_C(1109)) {
                                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        if (m < INT64_C(555)) {
                                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (m < INT64_C(1109)) {
                                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    }
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    if (n < INT64_C(124)) {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(2218)) {
                                                        select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(1109)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            } else {
                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(28)) {
                        if (m < INT64_C(17740)) {
                            if (k < INT64_C(56)) {
                                select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                return out;
                            } else {
                                if (k < INT64_C(118)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(35480)) {
                                select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(118)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(91)) {
                                if (n < INT64_C(46)) {
                                    if (k < INT64_C(63)) {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(167)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(222)) {
                                    if (k < INT64_C(363)) {
                                        if (k < INT64_C(91)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(97)) {
                                if (k < INT64_C(42)) {
                                    if (m < INT64_C(35480)) {
                                        if (k < INT64_C(20)) {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(26)) {
                                            select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(35480)) {
                                        select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(128)) {
                                            select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(4435)) {
                    if (m < INT64_C(2218)) {
                        if (k < INT64_C(287)) {
                            if (k < INT64_C(111)) {
                                if (m < INT64_C(784)) {
                                    if (k < INT64_C(79)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(992)) {
                                    if (k < INT64_C(203)) {
                                        if (m < INT64_C(139)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(278)) {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(555)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(1109)) {
                                                        if (k < INT64_C(144)) {
                                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(555)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(1620)) {
                                if (m < INT64_C(70)) {
                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(448)) {
                                        if (m < INT64_C(278)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(405)) {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(725)) {
                                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(725)) {
                                    if (m < INT64_C(139)) {
                                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            select_tf32_tn_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(139)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(393)) {
                                                select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                                return out;
                                            } else {
                                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(182)) {
                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(363)) {
                                if (n < INT64_C(725)) {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(182)) {
                            select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                            return out;
                        } else {
                            select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (k < INT64_C(291)) {
                if (n < INT64_C(23)) {
                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                    return out;
                } else {
                    select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                }
            } else {
                if (n < INT64_C(91)) {
                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                }
            }
        }
    } else {
        if (m < INT64_C(1792)) {
            if (n < INT64_C(2024)) {
                if (m < INT64_C(555)) {
                    if (m < INT64_C(6)) {
                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        if (m < INT64_C(70)) {
                            if (k < INT64_C(2897)) {
                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(28)) {
                                    select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(139)) {
                                select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                if (n < INT64_C(363)) {
                                    select_tf32_tn_config out = {2u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(278)) {
                                        if (k < INT64_C(3072)) {
                                            select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                        return out;
                                    }
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(1109)) {
                        if (k < INT64_C(2173)) {
                            select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(363)) {
                                select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (n < INT64_C(363)) {
                            if (k < INT64_C(1630)) {
                                select_tf32_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {2u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(12)) {
                    select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(10138)) {
                        select_tf32_tn_config out = {2u, 1u, 8u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(182)) {
                if (m < INT64_C(35480)) {
                    if (m < INT64_C(8870)) {
                        select_tf32_tn_config out = {1u, 1u, 4u, 16u, 16u};
                        return out;
                    } else {
                        select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_tn_config out = {8u, 2u, 4u, 16u, 16u};
                    return out;
                }
            } else {
                if (m < INT64_C(7168)) {
                    if (n < INT64_C(363)) {
                        if (m < INT64_C(4435)) {
                            if (k < INT64_C(1630)) {
                                select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {2u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(1630)) {
                                select_tf32_tn_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(3584)) {
                            if (m < INT64_C(3104)) {
                                select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                                return out;
                            } else {
                                select_tf32_tn_config out = {8u, 1u, 8u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                            return out;
                        }
                    }
                } else {
                    select_tf32_tn_config out = {4u, 2u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_TF32_TN_H */
